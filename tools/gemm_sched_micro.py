"""Schedules of the tcgen05 GEMM on weight-streaming (small-M) shapes:
1 = whole tiles, 2 = stream-K ranges, 3 = whole-tile waves + K-split tail
(for one token tile: every tile K-split). Weights rotate over 4 copies so each
launch streams from HBM."""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

_lib.call("sx_gemm_set_pair_mode", 1)
for (M, N, Kd, dual) in [(2, 4096, 4096, False), (2, 12288, 4096, False), (2, 11008, 4096, True),
                         (64, 4096, 4096, False), (64, 4096, 32768, False), (256, 4096, 4096, False),
                         (256, 4096, 11008, False), (256, 12288, 4096, False)]:
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    ws = [(torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() for _ in range(4)]
    w2s = [(torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() for _ in range(4)] if dual else [None] * 4
    epi = K.EPI_SWIGLU_BF16 if dual else K.EPI_BF16
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    line = []
    for sched in (1, 2, 3):
        for i in range(3):
            K.gemm(x, ws[i % 4], out=out, epi=epi, w2=w2s[i % 4], splits=sched)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for i in range(12):
            K.gemm(x, ws[i % 4], out=out, epi=epi, w2=w2s[i % 4], splits=sched)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / 12 * 1e3
        gbs = N * Kd * 2 * (2 if dual else 1) / (us * 1e3)
        line.append(f"s{sched} {us:7.1f}us {gbs:6.0f}GB/s plan={K.gemm_plan(M, N, Kd, dual, sched)[:2]}")
    print(f"M={M:4d} N={N:6d} K={Kd:6d} dual={int(dual)}: " + " | ".join(line))
    del x, ws, w2s, out
    torch.cuda.empty_cache()
