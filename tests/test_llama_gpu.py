"""Llama-shaped path on the GPU: logits vs the fp32 CPU reference (bf16
tolerance 2e-2 abs, north_star), tree-masked target pass vs full-prefix
recomputation, KV compaction, and bit-exact replay parity of the tree /
accepted tokens against the CPU oracle fed the GPU's own logits rows."""

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import llama_ref
from oracle import speckit_oracle as ox
from paper_2406_02532_b200.llama import PRESETS, LlamaModel, SyntheticBias

pytestmark = pytest.mark.gpu
TOL = 2e-2


def ref_logits(model, prefix):
    W = model.w.to_cpu_fp32()
    bias = None
    if model.synthetic is not None:
        bias = (model.bias_u.float().cpu(), model.bias_w.float().cpu())
    return llama_ref.forward_logits(model.cfg, W, list(prefix), bias)


@pytest.fixture(scope="module")
def pair():
    torch.cuda.set_device(0)
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    target = LlamaModel("tiny", seed=1, max_ctx=2048, max_tokens=512, synthetic=syn)
    draft = LlamaModel("tiny-draft", seed=2, max_ctx=4096, max_tokens=512, synthetic=syn)
    return draft, target


def test_prefix_logits_vs_cpu_reference(pair):
    draft, target = pair
    rng = np.random.default_rng(0)
    for m in (target, draft):
        for n in (1, 5, 37, 130):
            prefix = tuple(int(t) for t in rng.integers(0, 32000, size=n))
            got = m.prefix_rows(prefix)[0].cpu()
            exp = ref_logits(m, prefix)[-1]
            assert (got - exp).abs().max().item() < TOL, (m.cfg.name, n)


def test_tree_pass_rows_match_full_prefix(pair):
    draft, target = pair
    prompt = tuple(range(100, 140))
    tree = sx.build_sssp(prompt, draft, sx.BuilderParams(48, 6, 8), None)
    assert len(tree.nodes) == 48
    rows = target.tree_rows(tree).cpu()
    W = target.w.to_cpu_fp32()
    bias = (target.bias_u.float().cpu(), target.bias_w.float().cpu())
    # every node's row must equal a causal forward of its full prefix
    for node in tree.nodes[::3] + tree.nodes[-3:]:
        exp = llama_ref.forward_logits(target.cfg, W, list(tree.full_prefix(node.node_id)), bias)[-1]
        assert (rows[node.node_id + 1] - exp).abs().max().item() < TOL
    exp0 = llama_ref.forward_logits(target.cfg, W, list(prompt), bias)[-1]
    assert (rows[0] - exp0).abs().max().item() < TOL


def _replay_models(draft, target):
    """Oracle LogitsLMs serving the GPU's recorded rows, build by build."""
    state = {"k": -1}

    def make(recs):
        def fn(prefixes):
            tab = recs[state["k"]]
            return np.stack([tab[tuple(p)] for p in prefixes])

        return ox.LogitsLM(32000, fn)

    real = ox.precompute

    def pre(prefix, d, t, params, warp=None, warp_scores=True):
        state["k"] += 1
        return real(prefix, d, t, params, warp, warp_scores)

    return make(draft.record), make(target.record), pre


@pytest.mark.parametrize("t,p,warp_scores", [(0.0, 1.0, False), (0.0, 1.0, True), (0.6, 0.9, True)])
def test_engine_replay_parity(pair, monkeypatch, t, p, warp_scores):
    draft, target = pair
    draft.record, target.record = [], []
    prompt = tuple(int(x) for x in np.random.default_rng(5).integers(0, 32000, size=24))
    params = sx.BuilderParams(64, 8, 16)
    cfg = sx.SamplingConfig(t, p, seed=3, max_new_tokens=40)
    got, stats = sx.generate_specexec(prompt, draft, target, params, cfg, warp_scores=warp_scores)
    d_lm, t_lm, pre = _replay_models(draft, target)
    draft.record = target.record = None
    # the oracle rebuilds every tree and walk from the GPU's own rows
    monkeypatch.setattr(ox, "precompute", pre)
    exp, ostats = ox.generate_specexec(prompt, d_lm, t_lm, ox.BuilderParams(64, 8, 16),
                                       ox.SamplingConfig(t, p, seed=3, max_new_tokens=40), warp_scores=warp_scores)
    assert got == exp
    assert stats.accepted_per_iteration == ostats.accepted_per_iteration
    assert stats.draft_calls == ostats.draft_calls
    if warp_scores is False:
        assert stats.generation_rate > 1.0  # the synthetic correlation makes the draft useful


def test_tree_replay_bit_exact(pair):
    draft, target = pair
    draft.record = []
    prompt = tuple(range(7, 40))
    for warp in (None, sx.SamplingConfig(0.6, 0.9)):
        g = sx.build_sssp(prompt, draft, sx.BuilderParams(200, 10, 32), warp)
        tab = draft.record[-1]
        lm = ox.LogitsLM(32000, lambda ps: np.stack([tab[tuple(q)] for q in ps]))
        o = ox.build_sssp(prompt, lm, ox.BuilderParams(200, 10, 32), ox.SamplingConfig(0.6, 0.9) if warp else None)
        assert [(n.parent, n.token, n.edge_logprob, n.cum_logprob) for n in g.nodes] == \
            [(n.parent, n.token, n.edge_logprob, n.cum_logprob) for n in o.nodes]
        assert g.rounds == o.rounds
    draft.record = None


def test_kv_compaction_keeps_committed_prefix_exact(pair):
    draft, target = pair
    prompt = tuple(range(1000, 1030))
    cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=48)
    toks, stats = sx.generate_specexec(prompt, draft, target, sx.BuilderParams(96, 8, 16), cfg, warp_scores=False)
    assert len(toks) == 48 and len(stats.accepted_per_iteration) < 48
    full = prompt + tuple(toks)
    # rows served from the compacted KV cache == a causal recomputation on the CPU
    got = target.prefix_rows(full)[0].cpu()
    exp = ref_logits(target, full)[-1]
    assert (got - exp).abs().max().item() < TOL
    got_d = draft.prefix_rows(full)[0].cpu()
    exp_d = ref_logits(draft, full)[-1]
    assert (got_d - exp_d).abs().max().item() < TOL


def test_specexec_equals_sequential_greedy(pair):
    draft, target = pair
    prompt = tuple(range(500, 520))
    cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=32)
    got, _ = sx.generate_specexec(prompt, draft, target, sx.BuilderParams(64, 8, 16), cfg, warp_scores=False)
    seq, _ = sx.generate_sequential(prompt, target, cfg)
    assert got == seq


@pytest.mark.parametrize("nbuf", [2, 3, 8])
def test_offloaded_target_matches_resident(pair, nbuf):
    """Stage 3: the same weights streamed per layer from pinned host memory give
    bit-identical logits and tokens (same kernels, same order of operations),
    for a plain double buffer, a ring that does not divide the layer count and
    a ring deeper than the tiny model's layers (clamped)."""
    draft, _ = pair
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    res = LlamaModel("tiny", seed=11, max_ctx=2048, max_tokens=512, synthetic=syn)
    off = LlamaModel("tiny", seed=11, max_ctx=2048, max_tokens=512, synthetic=syn, offload=True, offload_buffers=nbuf)
    assert off.streamer.nbuf == min(nbuf, off.cfg.layers)
    prefix = tuple(range(300, 340))
    assert torch.equal(res.prefix_rows(prefix), off.prefix_rows(prefix))
    cfg = sx.SamplingConfig(0.6, 0.9, seed=5, max_new_tokens=30)
    a, sa = sx.generate_specexec((5, 6, 7, 8), draft, res, sx.BuilderParams(64, 8, 16), cfg)
    b, sb = sx.generate_specexec((5, 6, 7, 8), draft, off, sx.BuilderParams(64, 8, 16), cfg)
    assert a == b and sa.accepted_per_iteration == sb.accepted_per_iteration
    assert off.streamer.bytes >= off.w.layer_bytes * off.cfg.layers * sb.target_calls


@pytest.mark.parametrize("V,K_,D_,B_", [(128256, 2048, 8, 128), (32000, 8192, 12, 1024),
                                        # small budgets with batches wider than the tree (B > K): the
                                        # smallest merge-path sort (K = 48 -> 64) and the select path
                                        (32000, 48, 6, 256), (32000, 300, 8, 1024)])
def test_large_tree_replay_bit_exact(cuda, V, K_, D_, B_):
    """SURVEY 8(a) sizes: a Llama-3-vocabulary draft (V = 128256) and the largest
    budget (K = 8192) -- the GPU tree equals the oracle's build_sssp on the
    GPU's own rows (raw scoring), node for node."""
    from paper_2406_02532_b200.llama import LlamaConfig

    cfg = LlamaConfig(V, 256, 2, 2, 1, 512, 5e5, 1e-5, name=f"tiny-v{V}")
    draft = LlamaModel(cfg, seed=5, max_ctx=4 * K_ + 2 * B_ * (D_ + 1) + 256, max_tokens=max(B_, 64),
                       synthetic=SyntheticBias(seed=3, rank=64, scale=3.0))
    draft.record = []
    prompt = tuple(int(t) for t in np.random.default_rng(V + K_).integers(0, V, size=16))
    g = sx.build_sssp(prompt, draft, sx.BuilderParams(K_, D_, B_), None, warp_scores=False)
    tab = draft.record[-1]
    draft.record = None
    lm = ox.LogitsLM(V, lambda ps: np.stack([tab[tuple(q)] for q in ps]))
    o = ox.build_sssp(prompt, lm, ox.BuilderParams(K_, D_, B_), None, warp_scores=False)
    assert len(g.nodes) == min(K_, len(o.nodes)) and len(o.nodes) == K_
    assert [(n.parent, n.token) for n in g.nodes] == [(n.parent, n.token) for n in o.nodes]
    assert [n.edge_logprob for n in g.nodes] == [n.edge_logprob for n in o.nodes]
    assert g.rounds == o.rounds


def test_fused_qkv_rope_matches_separate_kernels(pair):
    """sx_gemm_qkv_rope (RoPE + KV scatter in the QKV GEMM epilogue, from the fp32
    accumulators) vs the separate GEMM (bf16 qkv) + rope_kv kernels: logits and
    cache rows agree to bf16 rounding."""
    _, target = pair
    prefix = tuple(int(t) for t in np.random.default_rng(42).integers(0, 32000, size=90))
    out = {}
    for fused in (False, True):
        target.fuse_rope = fused
        target.committed.clear()
        rows = target.prefix_rows(prefix)[0].clone()
        out[fused] = (rows, target.kc[:, :, : len(prefix) - 1].float().clone(),
                      target.vc[:, :, : len(prefix) - 1].float().clone())
    target.fuse_rope = True
    (ra, ka, va), (rb, kb, vb) = out[False], out[True]
    assert (ra - rb).abs().max().item() < TOL
    assert (ka - kb).abs().max().item() <= 2e-2 * max(1.0, ka.abs().max().item())
    assert (va - vb).abs().max().item() <= 2e-2 * max(1.0, va.abs().max().item())


@pytest.mark.parametrize("V,K_,B_", [(32000, 1024, 256), (128256, 512, 128)])
def test_fused_round_kernel_matches_two_kernel_path(cuda, V, K_, B_):
    """sx_tree_set_impl A/B: the chunked logits-row path (max / sum / score
    kernels over (row, chunk) units, one HBM read per prefiltered row) and the
    tree_row_stats + tree_score pair build the same tree, node for node, on the
    same draft rows."""
    from paper_2406_02532_b200 import _lib
    from paper_2406_02532_b200.llama import LlamaConfig

    cfg = LlamaConfig(V, 256, 2, 2, 1, 512, 1e4, 1e-5, name=f"fused-v{V}")
    draft = LlamaModel(cfg, seed=9, max_ctx=4 * K_ + 2 * B_ * 13 + 256, max_tokens=max(B_, 64),
                       synthetic=SyntheticBias(seed=4, rank=64, scale=3.0))
    prompt = tuple(int(t) for t in np.random.default_rng(V).integers(0, V, size=12))
    trees = []
    for impl in (1, 0):
        _lib.call("sx_tree_set_impl", impl)
        try:
            draft.committed.clear()
            g = sx.build_sssp(prompt, draft, sx.BuilderParams(K_, 12, B_), None, warp_scores=False)
            trees.append(([(n.parent, n.token, n.edge_logprob) for n in g.nodes], g.rounds))
        finally:
            _lib.call("sx_tree_set_impl", 0)
    assert trees[0] == trees[1]
