"""Max / mean abs error of both attention kernels vs the fp32 torch reference
(tests/test_attention_gpu.py helpers) on tree-pass shapes."""
import importlib.util
import pathlib
import sys

import numpy as np
import torch

root = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(root))
spec = importlib.util.spec_from_file_location("tattn", root / "tests" / "test_attention_gpu.py")
T = importlib.util.module_from_spec(spec)
spec.loader.exec_module(T)

rng = np.random.default_rng(5)
for H, KVH, N, ctx, D in [(64, 8, 1025, 130, 16), (32, 32, 1024, 160, 16), (64, 8, 1025, 1024, 1), (64, 8, 1025, 130, 1)]:
    paths = T.random_tree(rng, N, D)
    A = D + 1
    anc = np.zeros((N, A), np.int32)
    alen = np.zeros(N, np.int32)
    for t, pth in enumerate(paths):
        anc[t, : len(pth)] = pth
        alen[t] = len(pth)
    q, kc, vc = T.make(N, H, KVH, ctx + N + 8, seed=N)
    q = (q.float() * 3).bfloat16()  # sharper softmax than unit-variance scores
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    exp = T.reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    for impl in (1, 2):
        got = T.run(impl, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, A)
        e = (got - exp).abs()
        print(f"H={H} KVH={KVH} N={N} ctx={ctx} D={D} impl={impl}: max {float(e.max()):.3e} mean {float(e.mean()):.3e} "
              f"(ref rms {float(exp.pow(2).mean().sqrt()):.3f})", flush=True)
