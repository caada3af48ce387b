"""Multi-process host logic of bench.py (world_size 2, gloo, CPU): the timed
value is the MAX of per-rank device times and the token count is the SUM over
ranks (replicas, weak scaling)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ms = [120.0, 180.0][rank]
    toks = [7, 11][rank]
    out[rank] = (bench.max_over_ranks(ms, world, "cpu"), bench.sum_over_ranks(toks, world, "cpu"))
    bench.barrier(world)
    dist.destroy_process_group()


def test_replica_timing_reduction():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1] == (180.0, 18.0)
