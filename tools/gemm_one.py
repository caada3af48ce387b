"""Launch one GEMM shape a few times (for ncu captures): python tools/gemm_one.py SHAPE MODE [ITERS]"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2406_02532_b200 import _lib  # noqa: E402
from paper_2406_02532_b200 import kernels as K  # noqa: E402
from tools.gemm_bench import SHAPES  # noqa: E402

name, mode = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
_lib.call("sx_gemm_set_pair_mode", mode)
_, M, N, Kd, dual, epi = next(s for s in SHAPES if s[0] == name)
x = torch.randn(M, Kd, device="cuda").bfloat16()
w = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16()
w2 = (torch.randn(N, Kd, device="cuda") * 0.02).bfloat16() if dual else None
dt = torch.float32 if epi in (K.EPI_F32, K.EPI_ADD_F32) else torch.bfloat16
out = torch.zeros(M, N, dtype=dt, device="cuda")
for _ in range(iters):
    K.gemm(x, w, out=out, epi=epi, w2=w2)
torch.cuda.synchronize()
print("done", name, mode)
