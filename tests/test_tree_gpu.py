"""Stage 1 (GPU build_sssp) and stage 4 (GPU walk) parity on exact table models.

GPU vs CPU oracle: bit-exact -- identical parents, tokens, float64 edge /
cumulative log-probs and round counts (the kernels and oracle/oxmath.c share the
canonical arithmetic). GPU vs reference fixtures: identical topology, rounds,
tokens and stats (values within the oracle's pinned 1e-12).
"""

import json
import pathlib

import numpy as np
import pytest

import paper_2406_02532_b200 as sx
from oracle import speckit_oracle as ox

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())["data"]


def assert_same_tree(g, o, ctx=""):
    assert [n.parent for n in g.nodes] == [n.parent for n in o.nodes], ctx
    assert [n.token for n in g.nodes] == [n.token for n in o.nodes], ctx
    assert [n.edge_logprob for n in g.nodes] == [n.edge_logprob for n in o.nodes], ctx
    assert [n.cum_logprob for n in g.nodes] == [n.cum_logprob for n in o.nodes], ctx
    assert g.rounds == o.rounds, ctx


def warp_cfg(w, gpu=True):
    if not w:
        return None
    return (sx.SamplingConfig if gpu else ox.SamplingConfig)(*w, seed=0)


def test_worked_examples(cuda):
    tree = sx.build_sssp((), sx.TabularModel([0.6, 0.3, 0.1]), sx.BuilderParams(5, 2, 4))
    assert {tree.path_tokens(n.node_id) for n in tree.nodes} == {(0,), (0, 0), (1,), (0, 1), (1, 0)}
    chain = sx.MarkovModel(np.roll(np.eye(3), 1, axis=1), order=1)
    tree = sx.build_sssp((0,), chain, sx.BuilderParams(8, 4, 4))
    assert [tree.path_tokens(n.node_id) for n in tree.nodes] == [(1,), (1, 2), (1, 2, 0), (1, 2, 0, 1)]


def test_golden_tree(cuda):
    g = load("golden_tree.json")
    tree = sx.build_sssp(tuple(g["prefix"]), sx.make_synthetic(*g["model"]), sx.BuilderParams(*g["params"]),
                         sx.SamplingConfig(*g["warp"]))
    ref = g["dump"]["nodes"]
    assert [n.parent for n in tree.nodes] == [r["parent"] for r in ref]
    assert [n.token for n in tree.nodes] == [r["token"] for r in ref]
    for n, r in zip(tree.nodes, ref):
        assert abs(n.edge_logprob - r["edge_logprob"]) < 1e-12


def test_sssp_instances_vs_oracle_and_reference(cuda):
    data = load("sssp_instances.json")
    for inst in data["random"]:
        params = (inst["budget"], inst["depth"], inst["batch"])
        g = sx.build_sssp(tuple(inst["prompt"]), sx.make_synthetic(inst["model_seed"], inst["vocab"], inst["sharpness"]),
                          sx.BuilderParams(*params), warp_cfg(inst["warp"]))
        o = ox.build_sssp(tuple(inst["prompt"]), ox.make_synthetic(inst["model_seed"], inst["vocab"], inst["sharpness"]),
                          ox.BuilderParams(*params), warp_cfg(inst["warp"], gpu=False))
        assert_same_tree(g, o, inst)
        ref = inst["tree"]
        assert [n.parent for n in g.nodes] == ref["parent"] and [n.token for n in g.nodes] == ref["token"]
        assert g.rounds == ref["rounds"]


def test_uniform_ties_and_batch_invariance(cuda):
    uni = [0.25] * 4
    for K_, D_, B_ in [(25, 4, 4), (7, 3, 2), (40, 5, 16), (100, 6, 1)]:
        g = sx.build_sssp((1,), sx.TabularModel(uni), sx.BuilderParams(K_, D_, B_))
        o = ox.build_sssp((1,), ox.TabularModel(uni), ox.BuilderParams(K_, D_, B_))
        assert_same_tree(g, o, (K_, D_, B_))
    for i in range(10):
        m = sx.make_synthetic(300 + i, 7, 0.4)
        topo = None
        for B_ in (1, 2, 4, 16, 64):
            t = sx.build_sssp((2,), m, sx.BuilderParams(40, 5, B_), sx.SamplingConfig(0.6, 0.9))
            cur = [(n.parent, n.token) for n in t.nodes]
            assert topo is None or cur == topo
            topo = cur


def test_large_budget_markov_vs_oracle(cuda):
    # bigger trees: V=32 Markov, K up to 2048, several warps
    for seed, K_, D_, B_, w in [(1, 512, 16, 32, None), (2, 2048, 12, 64, (0.6, 0.9)), (3, 300, 16, 8, (0.0, 1.0)),
                                (4, 1024, 10, 128, (1.0, 0.8))]:
        g = sx.build_sssp((5, 7), sx.make_synthetic(seed, 32, 0.2), sx.BuilderParams(K_, D_, B_), warp_cfg(w))
        o = ox.build_sssp((5, 7), ox.make_synthetic(seed, 32, 0.2), ox.BuilderParams(K_, D_, B_), warp_cfg(w, False))
        assert_same_tree(g, o, (seed, K_, w))


def test_deep_narrow_trees_vs_oracle(cuda):
    # long ancestor chains (max_depth up to 250: the next-batch walk, the KV-slot
    # lists and the lex merge over many depths) and small batches (many rounds)
    for seed, V_, sharp, K_, D_, B_, w in [(21, 8, 0.02, 400, 200, 4, None), (22, 6, 0.05, 600, 250, 2, (0.6, 0.9)),
                                           (23, 16, 0.03, 1000, 120, 8, None)]:
        g = sx.build_sssp((3,), sx.make_synthetic(seed, V_, sharp), sx.BuilderParams(K_, D_, B_), warp_cfg(w))
        o = ox.build_sssp((3,), ox.make_synthetic(seed, V_, sharp), ox.BuilderParams(K_, D_, B_), warp_cfg(w, False))
        assert_same_tree(g, o, (seed, K_, D_, B_))
        assert max(n.depth for n in g.nodes) > 15  # the chains really are deep


def test_engine_grid_vs_reference(cuda):
    data = load("engine_grid.json")
    models = {}
    for rec in data["grid"]:
        i = rec["i"]
        if i not in models:
            models[i] = (sx.make_synthetic(2 * i, 10, 0.3), sx.make_synthetic(2 * i + 1, 10, 0.3))
        draft, target = models[i]
        cfg = sx.SamplingConfig(rec["t"], rec["top_p"], seed=i, max_new_tokens=16)
        got, stats = sx.generate_specexec(tuple(rec["prompt"]), draft, target, sx.BuilderParams(12, 5, 4), cfg)
        seq, _ = sx.generate_sequential(tuple(rec["prompt"]), target, cfg)
        assert got == rec["specexec"] == seq, rec
        assert stats.target_calls == rec["target_calls"] and stats.draft_calls == rec["draft_calls"]
        assert stats.accepted_per_iteration == rec["accepted"]


def test_demo03_c1(cuda):
    demo = load("engine_grid.json")["demo03"]
    target = sx.make_synthetic(*demo["model"])
    draft = target.power_smoothed(demo["draft_power"])
    for run in demo["runs"]:
        cfg = sx.SamplingConfig(run["t"], run["top_p"], seed=0, max_new_tokens=64)
        got, stats = sx.generate_specexec(tuple(demo["prompt"]), draft, target,
                                          sx.BuilderParams(demo["K"], demo["D"], demo["B"]), cfg)
        assert got == run["tokens"]
        assert stats.target_calls == run["target_calls"] and stats.draft_calls == run["draft_calls"]
        assert stats.accepted_per_iteration == run["accepted"]


def test_warp_and_sample_kernels_vs_oracle(cuda):
    import torch

    from paper_2406_02532_b200 import kernels as K

    rng = np.random.default_rng(0)
    for V in (3, 8, 300, 4096, 32000):
        for T, P in [(0.0, 1.0), (0.6, 0.9), (1.0, 0.5), (1.7, 1.0), (0.3, 0.99)]:
            z = (rng.standard_normal(V) * 3).astype(np.float32)
            p = rng.dirichlet(np.full(V, 0.3))
            gz = K.warp_rows(torch.tensor(z[None]).cuda(), T, P)[0].cpu().numpy()
            oz = ox.apply_warp(ox.softmax_row(z), ox.SamplingConfig(T, P))
            assert np.array_equal(gz, oz), (V, T, P)
            gp = K.warp_rows(torch.tensor(p[None]).cuda(), T, P)[0].cpu().numpy()
            op = ox.apply_warp(p, ox.SamplingConfig(T, P))
            assert np.array_equal(gp, op), (V, T, P, "probs")
            us = rng.random(4)
            got = K.sample_rows(torch.tensor(np.stack([gp] * 4)).cuda(), us).tolist()
            exp = [int(ox.lib().ox_sample(ox._dptr(np.ascontiguousarray(op)), V, float(u))) for u in us]
            assert got == exp
        sm = K.softmax_rows(torch.tensor(z[None]).cuda())[0].cpu().numpy()
        assert np.array_equal(sm, np.asarray(ox.softmax_row(z)))


def test_fault_injection_detected(cuda, monkeypatch):
    from paper_2406_02532_b200 import engine

    real = engine.precompute

    def corrupted(prefix, draft, target, params, warp=None):
        cache = real(prefix, draft, target, params, warp)
        if len(cache.tree.nodes) > 1:
            cache.dists[2] = cache.dists[1]
        return cache

    monkeypatch.setattr(engine, "precompute", corrupted)
    diverged = 0
    for i in range(10):
        draft, target = sx.make_synthetic(101 + 2 * i, 16, 0.3), sx.make_synthetic(102 + 2 * i, 16, 0.3)
        cfg = sx.SamplingConfig(0.6, 0.9, seed=i, max_new_tokens=24)
        got, _ = sx.generate_specexec((1, 2, 3, 4), draft, target, sx.BuilderParams(16, 6, 4), cfg)
        seq, _ = sx.generate_sequential((1, 2, 3, 4), target, cfg)
        diverged += got != seq
    assert diverged > 0


def _with_survivor_cap(cap, fn):
    from paper_2406_02532_b200 import _lib
    from paper_2406_02532_b200.models import _WS

    _WS._tls.ws = {}
    _lib.call("sx_tree_set_survivor_cap", cap)
    try:
        return fn(_WS)
    finally:
        _lib.call("sx_tree_set_survivor_cap", 0)
        _WS._tls.ws = {}


@pytest.mark.parametrize("seed,K_,D_,B_,w", [(11, 512, 8, 64, None), (12, 300, 10, 32, (0.6, 0.9)), (13, 200, 6, 16, (0.0, 1.0))])
def test_survivor_overflow_sliced_retry_vs_oracle(cuda, seed, K_, D_, B_, w):
    """A survivor buffer of V entries overflows on most rounds of a V = 32 Markov
    build: the round is re-run in row slices (merge-only updates, batch remapped,
    the last slice picks the next batch) and the tree still equals the oracle's,
    node for node and round for round."""
    def run(WS):
        g = sx.build_sssp((5, 7), sx.make_synthetic(seed, 32, 0.05), sx.BuilderParams(K_, D_, B_), warp_cfg(w))
        return g, WS.get(K_, B_, 32, D_).overflow_retries

    g, retries = _with_survivor_cap(32, run)
    o = ox.build_sssp((5, 7), ox.make_synthetic(seed, 32, 0.05), ox.BuilderParams(K_, D_, B_), warp_cfg(w, False))
    assert_same_tree(g, o, (seed, K_, w))
    if w != (0.0, 1.0):  # argmax scoring yields one candidate per row: never overflows
        assert retries > 0
