"""Per-k-block cycles of the single-CTA vs CTA-pair kernels with TMA disabled
after the ring fill (SX_GEMM_DEBUG=1), one tile per SM (pair: per SM pair), K=16384."""
import pathlib
import subprocess
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

Kd = 16384
for mode in (1, 2):
    _lib.call("sx_gemm_set_pair_mode", mode)
    for bn in (64, 128, 256):
        M, N = bn, 148 * 128
        x = torch.randn(M, Kd, device="cuda").bfloat16()
        w = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16()
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for _ in range(2):
            K.gemm(x, w, out=out, splits=1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            K.gemm(x, w, out=out, splits=1)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        kb = Kd // 64
        cyc = ms * 1e-3 * 1.965e9 / kb
        print(f"mode={mode} BN={bn:3d} {2 * M * N * Kd / ms / 1e9:7.1f} TFLOP/s  {cyc:6.0f} cyc/k-block per SM-tile")
        del x, w, out
