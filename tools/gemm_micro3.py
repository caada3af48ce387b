"""Single vs CTA-pair tcgen05 GEMM vs cuBLAS (torch.matmul, reference only) on
target-pass shapes, with and without data movement (SX_GEMM_DEBUG=1 skips TMA)."""
import os
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402


def t(fn, n=5):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


dbg = os.environ.get("SX_GEMM_DEBUG", "0")
for (M, N, Kd) in [(1025, 10240, 8192), (1280, 18944, 8192), (1024, 28672, 8192)]:
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16()
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fl = 2 * M * N * Kd
    res = []
    for mode in (1, 2):
        _lib.call("sx_gemm_set_pair_mode", mode)
        ms = t(lambda: K.gemm(x, w, out=out, splits=1))
        res.append(f"{['', 'single', 'pair'][mode]} {fl / ms / 1e9:6.0f}")
    if dbg == "0":
        ms = t(lambda: torch.matmul(x, w.t(), out=out))
        res.append(f"cublas {fl / ms / 1e9:6.0f}")
    print(f"debug={dbg} M={M} N={N} K={Kd} TFLOP/s: " + "  ".join(res))
