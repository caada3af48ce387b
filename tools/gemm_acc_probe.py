"""fp32-accumulation accuracy of the tcgen05 GEMM at the draft/target shapes:
GPU out vs the fp32 CPU product of the same bf16 operands (relative to the
output scale), per epilogue. GPU tool (not a test)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_02532_b200 import kernels as K  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    rep = []
    for M, N, Kd in [(1, 4096, 4096), (37, 4096, 4096), (1, 4096, 11008), (1, 22016, 4096), (1025, 8192, 8192),
                     (1, 32000, 4096)]:
        x = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
        w = (torch.randn(N, Kd, device="cuda", generator=g) * 0.02).bfloat16()
        out = K.gemm(x, w, epi=K.EPI_F32)
        ref = x.float().cpu() @ w.float().cpu().t()
        d = (out.cpu() - ref).abs()
        rep.append({"M": M, "N": N, "K": Kd, "max_abs": float(d.max()), "rel": float(d.max() / ref.abs().max()),
                    "mean_rel": float(d.mean() / ref.abs().mean())})
    print(json.dumps(rep, indent=1))


main()
