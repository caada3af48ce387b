"""Tensor-parallel partition of the target forward (tp.py), checked on CPU with
world_size 2 (gloo): every rank slices the same seeded fp32 weights with
TPShard.shard, runs the TP restatement of the forward (two all-reduces per
layer, all-gathered vocab-parallel logits) and must reproduce the unsharded
forward's logits on every rank. The GPU path uses the same TPShard slices
(tests/test_tp_gpu.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_02532_b200.llama import LlamaConfig
from paper_2406_02532_b200.tp import TPShard

CFG = LlamaConfig(vocab=96, d=64, layers=2, heads=4, kv_heads=2, ff=96, rope_theta=1e4, eps=1e-5, head_dim=16,
                  name="tp-test")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(cfg, seed=0):
    g = torch.Generator().manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=g) * 0.2  # noqa: E731
    hd = cfg.head_dim
    layers = []
    for _ in range(cfg.layers):
        layers.append({"wqkv": r((cfg.heads + 2 * cfg.kv_heads) * hd, cfg.d), "wo": r(cfg.d, cfg.heads * hd),
                       "wg": r(cfg.ff, cfg.d), "wu": r(cfg.ff, cfg.d), "wd": r(cfg.d, cfg.ff),
                       "n1": 1 + 0.1 * r(cfg.d), "n2": 1 + 0.1 * r(cfg.d)})
    return {"emb": r(cfg.vocab, cfg.d), "layers": layers, "nf": 1 + 0.1 * r(cfg.d), "lm": r(cfg.vocab, cfg.d)}


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import llama_ref

    sh = TPShard(rank, world)
    sh.check(CFG)
    W = _weights(CFG)
    Wl = {"emb": W["emb"], "nf": W["nf"], "lm": sh.shard(CFG, "lm", W["lm"]),
          "layers": [{k: sh.shard(CFG, k, v) for k, v in L.items()} for L in W["layers"]]}

    def gather(t):
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t.contiguous())
        return parts

    toks = [3, 17, 5, 90, 41, 41, 7]
    got = llama_ref.forward_logits_tp(CFG, Wl, toks, sh, dist.all_reduce, gather)
    exp = llama_ref.forward_logits(CFG, W, toks)
    out[rank] = float((got - exp).abs().max())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_partition_reproduces_unsharded_forward(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] < 1e-4, out[r]


def test_tp_shard_checks():
    with pytest.raises(ValueError):
        TPShard(0, 3).check(CFG)  # 3 does not divide 4 heads
    sh = TPShard(1, 2)
    assert sh.heads(CFG) == (2, 4) and sh.kv_heads(CFG) == (1, 2) and sh.vocab(CFG) == (48, 96)
    shapes = sh.local_shapes(CFG)
    assert shapes["wqkv"] == ((2 + 2) * 16, 64) and shapes["wd"] == (64, 48)


def _comm_worker(rank, world, port, out):
    """NcclComm (the torch.distributed communicator the GPU model uses) over
    gloo: all-reduce and the vocab-parallel logits gather + interleave."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_02532_b200.tp import NcclComm, gather_vocab

    comm = NcclComm()
    y = torch.full((3, 4), float(rank + 1))
    comm.all_reduce_(y)
    m, Vl = 5, 3
    full = torch.arange(m * Vl * world, dtype=torch.float32).view(m, Vl * world)
    local = full[:, rank * Vl : (rank + 1) * Vl].contiguous()
    got = torch.empty(m, Vl * world)
    gather_vocab(comm, local, got, torch.empty(world * m * Vl + 7))
    out[rank] = (float(y[0, 0]), bool(torch.equal(got, full)))
    dist.destroy_process_group()


def test_nccl_comm_semantics_over_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r][0] == 3.0 and out[r][1]
