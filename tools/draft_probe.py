"""Time one draft forward round in isolation (the draft half of a SpecExec
iteration, stage 1): n frontier tokens through the draft model with the tree
mask (committed prefix + a short ancestor list), per GEMM shape via the CUDA
event profiler, plus the whole round eager and as a CUDA graph.

  python tools/draft_probe.py [--model llama2-7b] [--rows 1,32,256,1024]
"""

import argparse
import json
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import kernels as Kern  # noqa: E402
from paper_2406_02532_b200.llama import PRESETS, LlamaModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-7b")
    ap.add_argument("--rows", default="1,32,256,1024")
    ap.add_argument("--ctx", type=int, default=160)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = [int(r) for r in a.rows.split(",")]
    nmax = max(rows)
    m = LlamaModel(a.model, seed=2, max_ctx=a.ctx + nmax + 64, max_tokens=max(nmax, a.ctx, 128))
    dev = m.device
    V = PRESETS[a.model].vocab
    # commit a prompt so the rows attend a real prefix
    prompt = torch.randint(0, V, (a.ctx,), dtype=torch.int32, device=dev)
    m.forward(a.ctx, prompt, None, 0, None, 0, torch.arange(1, a.ctx + 1, dtype=torch.int32, device=dev), 0,
              None, 0, None, 0, None)
    out = []
    for n in rows:
        tok = torch.randint(0, V, (n,), dtype=torch.int32, device=dev)
        pos = torch.full((n,), a.ctx, dtype=torch.int32, device=dev)
        slot = torch.arange(n, dtype=torch.int32, device=dev) + a.ctx
        dense = torch.full((n,), a.ctx - 1, dtype=torch.int32, device=dev)
        anc = torch.stack([torch.full((n,), a.ctx - 1, dtype=torch.int32, device=dev), slot], 1).contiguous()
        alen = torch.full((n,), 2, dtype=torch.int32, device=dev)

        def fwd():
            m.forward(n, tok, pos, 0, slot, 0, dense, 0, anc, 0, alen, 2, 0)

        for _ in range(3):
            fwd()
        torch.cuda.synchronize()
        Kern.PROFILER = Kern.GemmProfiler()
        fwd()
        shapes = Kern.PROFILER.by_shape(top=8)
        Kern.PROFILER = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            fwd()
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / a.iters
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fwd()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / a.iters
        rec = {"model": a.model, "rows": n, "eager_ms": round(eager, 4), "graph_ms": round(graph, 4),
               "gemm_ms": round(sum(s["ms_per_step"] for s in shapes), 4),
               "shapes": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()} for s in shapes]}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    if a.out:
        pathlib.Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in out))


if __name__ == "__main__":
    main()
