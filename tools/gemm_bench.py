"""Per-shape timing of the tcgen05 GEMM on the projections of the C2 workload
(Llama-2-70B target pass over K+1 = 1025 tree tokens; Llama-2-7B draft rounds at
B = 128 frontier nodes). CUDA events on the launching stream, 3 warm-up + 10
timed launches per shape; weights (the streamed operand) exceed L2 in total.

  python tools/gemm_bench.py [--mode 0|1|2] [--json out.json]
"""

import argparse
import json
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

DRAFT_M = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--draft-m=")), 128))
SHAPES = [
    # name, M (tokens), N (features), K, dual, epilogue
    ("70b.qkv", 1025, 10240, 8192, False, K.EPI_BF16),
    ("70b.o", 1025, 8192, 8192, False, K.EPI_F32),
    ("70b.gate_up", 1025, 28672, 8192, True, K.EPI_SWIGLU_BF16),
    ("70b.gate_up_il", 1025, 57344, 8192, False, K.EPI_SWIGLU_IL),
    ("70b.down", 1025, 8192, 28672, False, K.EPI_F32),
    ("70b.lm_head", 1025, 32000, 8192, False, K.EPI_F32),
    ("7b.qkv", DRAFT_M, 12288, 4096, False, K.EPI_BF16),
    ("7b.o", DRAFT_M, 4096, 4096, False, K.EPI_F32),
    ("7b.gate_up", DRAFT_M, 11008, 4096, True, K.EPI_SWIGLU_BF16),
    ("7b.gate_up_il", DRAFT_M, 22016, 4096, False, K.EPI_SWIGLU_IL),
    ("7b.down", DRAFT_M, 4096, 11008, False, K.EPI_F32),
    ("7b.lm_head", DRAFT_M, 32000, 4096, False, K.EPI_F32),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--json", default=None)
    ap.add_argument("--sched", type=int, default=0, help="1 = whole tiles, 0 = auto (stream-K when waves are uneven)")
    ap.add_argument("--draft-m", type=int, default=128, help="(use --draft-m=N: read at import)")
    ap.add_argument("--only", default="", help="shape-name prefix filter")
    a = ap.parse_args()
    _lib.call("sx_gemm_set_pair_mode", a.mode)
    res = []
    for name, M, N, Kd, dual, epi in SHAPES:
        if not name.startswith(a.only):
            continue
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        # several weight copies so consecutive launches stream from HBM, not L2
        ncopy = max(1, int(2e9 // (N * Kd * 2 * (2 if dual else 1))))
        ws = [(torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() for _ in range(min(ncopy, 4))]
        w2s = [(torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() for _ in range(len(ws))] if dual else None
        dt = torch.float32 if epi in (K.EPI_F32, K.EPI_ADD_F32) else torch.bfloat16
        out = torch.zeros(M, N, dtype=dt, device="cuda")
        for i in range(3):
            K.gemm(x, ws[i % len(ws)], out=out, epi=epi, w2=w2s[i % len(ws)] if dual else None, splits=a.sched)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        s.record()
        for i in range(n):
            K.gemm(x, ws[i % len(ws)], out=out, epi=epi, w2=w2s[i % len(ws)] if dual else None, splits=a.sched)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        flops = 2.0 * M * N * Kd * (2 if dual else 1)
        wbytes = N * Kd * 2 * (2 if dual else 1)
        r = {"shape": name, "M": M, "N": N, "K": Kd, "dual": dual, "ms": ms, "tflops": flops / ms / 1e9,
             "weight_gbs": wbytes / ms / 1e6, "plan": K.gemm_plan(M, N, Kd, dual, a.sched)}
        res.append(r)
        print(f"{name:14s} M={M:5d} N={N:6d} K={Kd:6d} {ms:8.3f} ms {r['tflops']:7.1f} TFLOP/s "
              f"{r['weight_gbs']:7.0f} GB/s(weights) plan(bn,splits,ws)={r['plan']}")
        del ws, w2s, x, out
        torch.cuda.empty_cache()
    if a.json:
        pathlib.Path(a.json).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
