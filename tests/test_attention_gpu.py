"""Tree attention (`sx_tree_attention`, csrc/attention.cu) against an fp32 torch
restatement of the flattened ancestor mask (pkg/src/speckit/tree.py:208-219):
query t sees KV slots [0, dense_len[t]) plus its ancestor list. Each kernel
forced (mma.sync, tcgen05) and the by-shape default, on GQA groups 1 / 4 / 8, tree passes,
causal prefill, one-token chains, empty rows and long contexts that move the
running max across tiles."""

import math

import numpy as np
import pytest
import torch

from paper_2406_02532_b200 import _lib

pytestmark = pytest.mark.gpu
p = _lib.ptr


def reference(q, kc, vc, dense, anc, alen, anc_base):
    N, H, D = q.shape
    KVH = kc.shape[0]
    G = H // KVH
    qf, kf, vf = q.float(), kc.float(), vc.float()
    out = torch.zeros(N, H, D, device=q.device)
    for t in range(N):
        keys = list(range(int(dense[t]))) + [anc_base + int(x) for x in anc[t, : int(alen[t])]]
        if not keys:
            continue
        idx = torch.tensor(keys, device=q.device)
        k, v = kf[:, idx], vf[:, idx]  # [KVH, n, D]
        s = torch.einsum("kgd,knd->kgn", qf[t].view(KVH, G, D), k) / math.sqrt(D)
        out[t] = torch.einsum("kgn,knd->kgd", torch.softmax(s, -1), v).reshape(H, D)
    return out


def random_tree(rng, n, max_depth):
    parent, depth = [-1], [0]
    for i in range(1, n):
        ok = [j for j in range(max(0, i - 64), i) if depth[j] < max_depth] or [0]
        par = ok[int(rng.integers(0, len(ok)))]
        parent.append(par)
        depth.append(depth[par] + 1)
    paths = []
    for i in range(n):
        path, x = [], i
        while x != -1:
            path.append(x)
            x = parent[x]
        paths.append(path[::-1])
    return paths


def run(impl, q, kc, vc, dense, dense_const, anc, alen, anc_base, A, split=True):
    """split: pass the key-split workspace (tcgen05 kernel on small grids)."""
    N, H, _ = q.shape
    KVH = kc.shape[0]
    out = torch.empty_like(q)
    nws = int(_lib.load().sx_tree_attention_ws_bytes(N, H, KVH)) if split else 0
    ws = torch.zeros(max(nws, 1), dtype=torch.uint8, device=q.device)  # arrival counters start at 0
    _lib.call("sx_attention_set_impl", impl)
    try:
        _lib.call("sx_tree_attention_ws", p(q), p(kc), p(vc), kc.shape[1], p(dense) if dense is not None else None,
                  dense_const, p(anc) if anc is not None else None, anc_base, p(alen) if alen is not None else None,
                  A, p(out), N, H, KVH, p(ws) if nws else None, nws, _lib.stream_ptr())
    finally:
        _lib.call("sx_attention_set_impl", 0)
    torch.cuda.synchronize()
    return out.float()


def make(N, H, KVH, slots, seed, kscale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn(N, H, 128, device="cuda", generator=g).bfloat16()
    kc = (torch.randn(KVH, slots, 128, device="cuda", generator=g) * kscale).bfloat16()
    vc = torch.randn(KVH, slots, 128, device="cuda", generator=g).bfloat16()
    return q, kc, vc


@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("H,KVH,N,ctx,D", [(64, 8, 1025, 130, 16), (32, 8, 300, 70, 16), (32, 32, 257, 200, 16),
                                           (64, 8, 37, 0, 5),
                                           # grids >= 148 CTAs with G <= 2 (MHA-like drafts): the
                                           # ancestors take the CUDA-core pass of the tcgen05 kernel
                                           (32, 32, 1024, 100, 16), (32, 16, 600, 64, 12), (16, 16, 1500, 0, 20)])
def test_tree_pass(cuda, impl, H, KVH, N, ctx, D):
    rng = np.random.default_rng(N + ctx)
    paths = random_tree(rng, N, D)
    A = D + 1
    anc = np.zeros((N, A), dtype=np.int32)
    alen = np.zeros(N, dtype=np.int32)
    for t, path in enumerate(paths):
        anc[t, : len(path)] = path
        alen[t] = len(path)
    q, kc, vc = make(N, H, KVH, ctx + N + 8, seed=N)
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    anc_t, alen_t = torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda()
    got = run(impl, q, kc, vc, dense, 0, anc_t, alen_t, ctx, A)
    exp = reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    torch.testing.assert_close(got, exp, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("H,KVH,N", [(64, 8, 128), (32, 32, 200), (32, 8, 1)])
def test_causal_prefill_and_chain(cuda, impl, H, KVH, N):
    base = 50 if N == 1 else 0  # one-token chain step at slot 50
    q, kc, vc = make(N, H, KVH, base + N + 4, seed=7 + N)
    dense = torch.arange(base + 1, base + N + 1, dtype=torch.int32, device="cuda")
    got = run(impl, q, kc, vc, dense, 0, None, None, 0, 0)
    exp = reference(q, kc, vc, dense.cpu(), np.zeros((N, 0), np.int32), np.zeros(N, np.int32), 0)
    torch.testing.assert_close(got, exp, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("impl", [0, 1, 2])
def test_empty_rows_and_dense_const(cuda, impl):
    N, H, KVH = 20, 16, 2
    q, kc, vc = make(N, H, KVH, 300, seed=3)
    # dense_const for all rows, ancestor lists of varying length (some empty)
    alen = np.array([i % 4 for i in range(N)], dtype=np.int32)
    anc = np.zeros((N, 3), dtype=np.int32)
    for t in range(N):
        anc[t, : alen[t]] = [(t * 7 + j) % 40 for j in range(alen[t])]
    got = run(impl, q, kc, vc, None, 90, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), 200, 3)
    exp = reference(q, kc, vc, [90] * N, anc, alen, 200)
    torch.testing.assert_close(got, exp, atol=2e-2, rtol=2e-2)
    # rows with no keys at all produce zeros
    dense0 = torch.zeros(N, dtype=torch.int32, device="cuda")
    z = run(impl, q, kc, vc, dense0, 0, torch.from_numpy(anc).cuda(), torch.zeros(N, dtype=torch.int32, device="cuda"),
            200, 3)
    assert torch.count_nonzero(z) == 0


@pytest.mark.parametrize("impl", [0, 1, 2])
def test_long_context_running_max(cuda, impl):
    """Keys grow in magnitude along the context, so the row max keeps rising
    across key tiles (exercises the lazy O rescale of the tcgen05 kernel)."""
    N, H, KVH, ctx = 17, 64, 8, 2000
    q, kc, vc = make(N, H, KVH, ctx + N, seed=11)
    ramp = torch.linspace(0.2, 3.0, ctx + N, device="cuda").view(1, -1, 1)
    kc = (kc.float() * ramp).bfloat16()
    q = (q.float() * 2).bfloat16()
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    anc = np.arange(N, dtype=np.int32).reshape(N, 1)
    alen = np.ones(N, dtype=np.int32)
    got = run(impl, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, 1)
    exp = reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    torch.testing.assert_close(got, exp, atol=2e-2, rtol=2e-2)


def test_tcgen05_error_matches_mma_sync(cuda):
    """The tcgen05 kernel is as accurate as the mma.sync loop against fp32
    (same bf16 P rounding; no lazy-max drift), on a sharp tree-pass softmax."""
    rng = np.random.default_rng(5)
    N, H, KVH, ctx, D = 1025, 64, 8, 130, 16
    paths = random_tree(rng, N, D)
    anc = np.zeros((N, D + 1), np.int32)
    alen = np.zeros(N, np.int32)
    for t, path in enumerate(paths):
        anc[t, : len(path)] = path
        alen[t] = len(path)
    q, kc, vc = make(N, H, KVH, ctx + N + 8, seed=N)
    q = (q.float() * 3).bfloat16()
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    exp = reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    err = {}
    for impl in (1, 2):
        got = run(impl, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, D + 1)
        err[impl] = (got - exp).abs()
    assert float(err[2].max()) <= 1.25 * float(err[1].max()) + 1e-3, (float(err[2].max()), float(err[1].max()))
    assert float(err[2].mean()) <= 1.1 * float(err[1].mean()) + 1e-5, (float(err[2].mean()), float(err[1].mean()))


def test_deep_ancestor_lists_mha(cuda):
    """MHA batch with 40-entry ancestor lists (max_depth 39): past the 64-row
    kernel's static ancestor capacity, so the by-shape choice must take the
    tcgen05 kernel (dynamic ancestor list) and still match the reference."""
    rng = np.random.default_rng(9)
    N, H, KVH, ctx, D = 200, 8, 8, 64, 39
    paths = random_tree(rng, N, D)
    A = D + 1
    anc = np.zeros((N, A), np.int32)
    alen = np.zeros(N, np.int32)
    for t, path in enumerate(paths):
        anc[t, : len(path)] = path
        alen[t] = len(path)
    q, kc, vc = make(N, H, KVH, ctx + N + 8, seed=4)
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    got = run(0, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, A)
    exp = reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    torch.testing.assert_close(got, exp, atol=2e-2, rtol=2e-2)
    with pytest.raises(ValueError):
        run(1, q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, A)


@pytest.mark.parametrize("H,KVH,N,ctx,D", [(64, 8, 1, 300, 0), (32, 32, 1, 700, 0), (64, 8, 37, 130, 16),
                                           (32, 32, 256, 160, 16), (32, 8, 200, 2000, 3)])
def test_key_split_matches_unsplit(cuda, H, KVH, N, ctx, D):
    """Small grids run the tcgen05 kernel with its key tiles split over several
    CTAs and merged by attn_combine_kernel: same result as one CTA per tile
    row (and as the fp32 reference)."""
    assert _lib.load().sx_tree_attention_ws_bytes(N, H, KVH) > 0
    rng = np.random.default_rng(N + ctx)
    A = D + 1
    anc = np.zeros((N, A), np.int32)
    alen = np.zeros(N, np.int32)
    if D > 0:
        for t, path in enumerate(random_tree(rng, N, D)):
            anc[t, : len(path)] = path
            alen[t] = len(path)
    else:
        alen[:] = 1
        anc[:, 0] = np.arange(N)
    q, kc, vc = make(N, H, KVH, ctx + N + 8, seed=N + 1)
    dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
    args = (q, kc, vc, dense, 0, torch.from_numpy(anc).cuda(), torch.from_numpy(alen).cuda(), ctx, A)
    got_split = run(2, *args, split=True)
    got_one = run(2, *args, split=False)
    exp = reference(q, kc, vc, dense.cpu(), anc, alen, ctx)
    torch.testing.assert_close(got_split, exp, atol=2e-2, rtol=2e-2)
    torch.testing.assert_close(got_split, got_one, atol=1e-2, rtol=1e-2)


def test_key_split_workspace_reused_across_shapes(cuda):
    """One zero-once workspace serves split launches of different grid sizes
    (the model's shared 'attn' scratch: draft buckets, one-token graphs, target
    passes). A small grid's partials must never land on a larger grid's arrival
    counters (fixed counter header, attention.cu kAttnCounterBytes)."""
    H, KVH, ctx = 64, 8, 600
    shapes = [1, 32, 200, 1, 100, 200]  # G = 8: 16 tokens per CTA -> 8..104 CTAs, all split
    nmax = max(int(_lib.load().sx_tree_attention_ws_bytes(n, H, KVH)) for n in shapes)
    ws = torch.zeros(nmax, dtype=torch.uint8, device="cuda")
    _lib.call("sx_attention_set_impl", 2)
    try:
        for i, N in enumerate(shapes):
            nws = int(_lib.load().sx_tree_attention_ws_bytes(N, H, KVH))
            assert nws > 0
            q, kc, vc = make(N, H, KVH, ctx + N + 8, seed=100 + i)
            dense = torch.full((N,), ctx, dtype=torch.int32, device="cuda")
            anc = torch.arange(N, dtype=torch.int32, device="cuda").view(N, 1)
            alen = torch.ones(N, dtype=torch.int32, device="cuda")
            out = torch.empty_like(q)
            _lib.call("sx_tree_attention_ws", p(q), p(kc), p(vc), kc.shape[1], p(dense), 0, p(anc), ctx, p(alen), 1,
                      p(out), N, H, KVH, p(ws), nmax, _lib.stream_ptr())
            torch.cuda.synchronize()
            exp = reference(q, kc, vc, dense.cpu(), anc.cpu().numpy(), alen.cpu().numpy(), ctx)
            torch.testing.assert_close(out.float(), exp, atol=2e-2, rtol=2e-2)
    finally:
        _lib.call("sx_attention_set_impl", 0)
