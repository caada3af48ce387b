"""Main-loop throughput of the tcgen05 GEMM with exactly one tile per SM (or
per CTA pair) and a long K, so waves, epilogue and launch overhead vanish."""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

Kd = 32768
for mode in (1, 2):
    _lib.call("sx_gemm_set_pair_mode", mode)
    for bn in (64, 128, 160, 192, 208, 224, 256):
        M = bn
        N = 148 * 128  # 148 single tiles or 74 pair tiles
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
        print(f"mode={mode} BN={bn:3d} {ms:7.3f} ms {2 * M * N * Kd / ms / 1e9:7.1f} TFLOP/s  "
              f"L2->SM {((M + N) * Kd * 2 * (148 if mode == 1 else 74) / 148) / ms / 1e9 if False else (N * Kd * 2 + (148 if mode == 1 else 74) * M * Kd * 2) / ms / 1e9:7.0f} GB/s")
        del x, w, out
