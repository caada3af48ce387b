"""The product's process-level tensor-parallel path (bench.py --gpus N):
`LlamaModel(tp=NcclComm())` in one process per rank over torch.distributed --
here two processes sharing the one GPU this run has, on a gloo group (NCCL
refuses two ranks on one device; NcclComm stages through host memory under
gloo, the same calls otherwise). Each rank holds its Megatron shard (tp.py);
the ranks must produce the unsharded model's logits (bf16 reductions, 2e-2),
identical rows on every rank, and identical SpecExec tokens equal to TP
greedy decoding."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2406_02532_b200 as sx
    from paper_2406_02532_b200.llama import LlamaConfig, LlamaModel
    from paper_2406_02532_b200.tp import NcclComm

    cfg = LlamaConfig(32000, 256, 2, 4, 2, 512, 1e4, 1e-5, name="tp2-test")
    comm = NcclComm()
    assert comm.world == world and comm.host_staging
    target = LlamaModel(cfg, seed=3, max_ctx=2048, max_tokens=256, tp=comm, tp_fused=False)
    draft = LlamaModel("tiny-draft", seed=4, max_ctx=4096, max_tokens=256)
    prompt = tuple(range(200, 240))
    rows = target.prefix_rows(prompt)[0].cpu()
    res = {"rows": rows}
    if rank == 0:
        full = LlamaModel(cfg, seed=3, max_ctx=2048, max_tokens=256)
        res["err_vs_unsharded"] = float((rows - full.prefix_rows(prompt)[0].cpu()).abs().max())
        del full
    cfg_s = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=20)
    res["spec"], st = sx.generate_specexec(prompt, draft, target, sx.BuilderParams(64, 8, 16), cfg_s, warp_scores=False)
    res["seq"], _ = sx.generate_sequential(prompt, target, cfg_s)
    res["accepted"] = st.accepted_per_iteration
    # KV1: argmax keys MAX-reduced over the ranks (host-staged under gloo) instead of gathered rows
    target_k = LlamaModel(cfg, seed=3, max_ctx=2048, max_tokens=256, tp=comm, tp_fused=False, tp_argmax=True)
    draft_k = LlamaModel("tiny-draft", seed=4, max_ctx=4096, max_tokens=256)
    res["spec_kv1"], _ = sx.generate_specexec(prompt, draft_k, target_k, sx.BuilderParams(64, 8, 16), cfg_s,
                                              warp_scores=False)
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_tp_target(cuda):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r0, r1 = out[0], out[1]
    assert r0["err_vs_unsharded"] < 2e-2, r0["err_vs_unsharded"]
    assert torch.equal(r0["rows"], r1["rows"])  # every rank holds the same all-reduced rows
    assert r0["spec"] == r1["spec"] == r0["seq"] == r1["seq"] == r0["spec_kv1"] == r1["spec_kv1"]
    assert r0["accepted"] == r1["accepted"]
