#!/bin/bash
mkdir -p gpurun_out
for at in mma auto; do
timeout 900 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 256,1024 --batch 1024 --methods sx --seeds 2 --tokens 48 --synthetic 4 --attn $at --out gpurun_out/acc_$at.jsonl > gpurun_out/acc_$at.log 2>&1
done
timeout 300 python - > gpurun_out/attn_err.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from tests import test_attention_gpu as T
rng = np.random.default_rng(5)
for H, KVH, N, ctx, D in [(64, 8, 1025, 130, 16), (32, 32, 1024, 160, 16), (64, 8, 1025, 1024, 1)]:
    paths = T.random_tree(rng, N, D); A = D + 1
    anc = np.zeros((N, A), np.int32); alen = np.zeros(N, np.int32)
    for t, pth in enumerate(paths):
        anc[t, :len(pth)] = pth; alen[t] = len(pth)
    q, kc, vc = T.make(N, H, KVH, ctx + N + 8, seed=N)
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    exp = T.reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    for impl in (1, 2):
        got = T.run(impl, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, A)
        e = (got - exp).abs()
        print(H, KVH, N, ctx, D, "impl", impl, "max", float(e.max()), "mean", float(e.mean()), "rms_ref", float(exp.pow(2).mean().sqrt()))
PY
