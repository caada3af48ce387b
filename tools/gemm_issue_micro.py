"""MMA issue-rate characterisation: SX_GEMM_DEBUG=1 (no TMA after the ring
fill), one token tile of width BN per SM, 148 tiles, K=16384; reports cycles per
k-block (4 x tcgen05.mma 128 x BN x 16) at the observed SM clock."""
import os
import pathlib
import subprocess
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402

Kd = 16384
for bn in (32, 64, 96, 128, 160, 208, 256):
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
    clk = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                               capture_output=True, text=True).stdout.strip() or 1965)
    kb = Kd // 64
    cyc = ms * 1e-3 * clk * 1e6 / kb
    ideal = 4 * 128 * bn * 16 / 4096  # cycles at 4096 MAC/clk/SM
    print(f"debug={os.environ.get('SX_GEMM_DEBUG', '0')} BN={bn:3d} {ms * 1e3:8.1f} us  {2 * M * N * Kd / ms / 1e9:7.1f} TFLOP/s"
          f"  {cyc:6.0f} cyc/k-block (MMA ideal {ideal:4.0f}) clk~{clk:.0f}")
    del x, w, out
