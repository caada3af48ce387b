"""The real 70B target-pass shapes with the GEMM's TMA disabled after the first
ring fill (SX_GEMM_DEBUG=1): measures the pure tcgen05 MMA + barrier rate of the
single-CTA kernel, to separate data movement from issue limits."""
import os
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

_lib.call("sx_gemm_set_pair_mode", 1)
for (M, N, Kd) in [(1025, 10240, 8192), (1025, 8192, 28672), (208 * 5, 148 * 128 // 5 * 5, 8192)]:
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
    print(f"debug={os.environ.get('SX_GEMM_DEBUG', '0')} M={M} N={N} K={Kd} {ms:7.3f} ms {2 * M * N * Kd / ms / 1e9:7.1f} TFLOP/s")
