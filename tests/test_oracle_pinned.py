"""Pin the CPU oracle to the reference: golden vectors produced by running the
reference itself (oracle/gen_fixtures.py) and the reference's worked examples.

Topology (parent ids, tokens), round counts, generated tokens and call stats
must match exactly; float64 log-probs may differ from numpy's SIMD log by a few
ulp (documented deviation, oracle/oxmath.c), so they are compared at 1e-12.
"""

import json
import math
import pathlib
import random
import struct

import numpy as np
import pytest

from oracle import speckit_oracle as ox

GOLD = pathlib.Path(__file__).parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())["data"]


def ulp_diff(a: float, b: float) -> int:
    ia = struct.unpack("<q", struct.pack("<d", a))[0]
    ib = struct.unpack("<q", struct.pack("<d", b))[0]
    return abs(ia - ib)


def assert_tree_matches(tree, rec, ctx):
    assert [n.parent for n in tree.nodes] == rec["parent"], ctx
    assert [n.token for n in tree.nodes] == rec["token"], ctx
    assert tree.rounds == rec["rounds"], ctx
    for n, e, c in zip(tree.nodes, rec["edge"], rec["cum"]):
        assert abs(n.edge_logprob - e) <= 1e-12 + 1e-14 * abs(e), ctx
        assert abs(n.cum_logprob - c) <= 1e-12 + 1e-14 * abs(c), ctx


def test_ox_log_exp_are_faithful():
    rng = random.Random(0)
    xs = [rng.uniform(1e-300, 1.0) for _ in range(20000)] + [10 ** rng.uniform(-300, 300) for _ in range(20000)]
    xs += [1.0, 0.5, 2.0, 1e-310, 5e-324, 0.9999999999999999, 1.0000000000000002]
    got = ox.ox_log(np.array(xs))
    worst = max(ulp_diff(g, math.log(x)) for g, x in zip(got.tolist(), xs) if x != 1.0)
    assert worst <= 1
    assert ox.ox_log(np.array([1.0]))[0] == 0.0
    assert ox.ox_log(np.array([0.0]))[0] == -math.inf
    ys = [rng.uniform(-745.0, 0.0) for _ in range(20000)] + [rng.uniform(-1, 1) for _ in range(20000)]
    got = ox.ox_exp(np.array(ys))
    worst = max(ulp_diff(g, math.exp(y)) for g, y in zip(got.tolist(), ys) if math.exp(y) > 1e-300)
    assert worst <= 1


def test_golden_tree_file():
    g = load("golden_tree.json")
    model = ox.make_synthetic(*g["model"])
    tree = ox.build_sssp(tuple(g["prefix"]), model, ox.BuilderParams(*g["params"]), ox.SamplingConfig(*g["warp"]))
    dump = g["dump"]
    assert [n.parent for n in tree.nodes] == [r["parent"] for r in dump["nodes"]]
    assert [n.token for n in tree.nodes] == [r["token"] for r in dump["nodes"]]
    for n, r in zip(tree.nodes, dump["nodes"]):
        assert abs(n.edge_logprob - r["edge_logprob"]) < 1e-12
        assert abs(n.cum_logprob - r["cum_logprob"]) < 1e-12


def test_worked_examples():
    # pkg/tests/test_tree.py:60-87
    tree = ox.build_sssp((), ox.TabularModel([0.6, 0.3, 0.1]), ox.BuilderParams(5, 2, 4))
    paths = {tree.path_tokens(n.node_id) for n in tree.nodes}
    assert paths == {(0,), (0, 0), (1,), (0, 1), (1, 0)}
    chain = ox.MarkovModel(np.roll(np.eye(3), 1, axis=1), order=1)
    tree = ox.build_sssp((0,), chain, ox.BuilderParams(8, 4, 4))
    assert [tree.path_tokens(n.node_id) for n in tree.nodes] == [(1,), (1, 2), (1, 2, 0), (1, 2, 0, 1)]


def test_sampling_worked_examples():
    # pkg/tests/test_sampling.py:18-42
    d = np.array([0.1, 0.2, 0.3, 0.4])
    assert np.array_equal(ox.apply_warp(d, ox.SamplingConfig(1.0, 1.0)), d)
    assert ox.apply_warp(np.array([0.4, 0.4, 0.2]), ox.SamplingConfig(0.0)).tolist() == [1.0, 0.0, 0.0]
    out = ox.apply_warp(np.array([0.5, 0.3, 0.2]), ox.SamplingConfig(1.0, 0.7))
    assert np.allclose(out, [0.625, 0.375, 0.0], atol=1e-12)
    assert ox.apply_warp(np.array([0.5, 0.3, 0.2]), ox.SamplingConfig(top_p=0.5)).tolist() == [1.0, 0.0, 0.0]


def test_sssp_instances_match_reference():
    data = load("sssp_instances.json")
    for inst in data["random"]:
        model = ox.make_synthetic(inst["model_seed"], inst["vocab"], inst["sharpness"])
        warp = ox.SamplingConfig(*inst["warp"], seed=0) if inst["warp"] else None
        tree = ox.build_sssp(tuple(inst["prompt"]), model, ox.BuilderParams(inst["budget"], inst["depth"], inst["batch"]), warp)
        assert_tree_matches(tree, inst["tree"], inst)
    for inst in data["extra"]:
        if inst["kind"] == "tabular":
            model = ox.TabularModel(inst["row"])
        else:
            model = ox.MarkovModel(np.roll(np.eye(3), 1, axis=1), order=1)
        tree = ox.build_sssp(tuple(inst["prompt"]), model, ox.BuilderParams(inst["budget"], inst["depth"], inst["batch"]))
        assert_tree_matches(tree, inst["tree"], inst)


def test_engine_grid_matches_reference():
    data = load("engine_grid.json")
    models = {}
    for rec in data["grid"]:
        i = rec["i"]
        if i not in models:
            models[i] = (ox.make_synthetic(2 * i, 10, 0.3), ox.make_synthetic(2 * i + 1, 10, 0.3))
        draft, target = models[i]
        cfg = ox.SamplingConfig(rec["t"], rec["top_p"], seed=i, max_new_tokens=16)
        got, stats = ox.generate_specexec(tuple(rec["prompt"]), draft, target, ox.BuilderParams(12, 5, 4), cfg)
        seq, _ = ox.generate_sequential(tuple(rec["prompt"]), target, cfg)
        assert got == rec["specexec"] and seq == rec["sequential"] and got == seq, rec
        assert stats.target_calls == rec["target_calls"] and stats.draft_calls == rec["draft_calls"]
        assert stats.accepted_per_iteration == rec["accepted"]


def test_demo03_c1_matches_reference():
    demo = load("engine_grid.json")["demo03"]
    target = ox.make_synthetic(*demo["model"])
    draft = target.power_smoothed(demo["draft_power"])
    for run in demo["runs"]:
        cfg = ox.SamplingConfig(run["t"], run["top_p"], seed=0, max_new_tokens=64)
        got, stats = ox.generate_specexec(tuple(demo["prompt"]), draft, target, ox.BuilderParams(demo["K"], demo["D"], demo["B"]), cfg)
        assert got == run["tokens"]
        assert stats.target_calls == run["target_calls"] and stats.draft_calls == run["draft_calls"]


def logits_lm(spec):
    bias = None
    if spec.get("bias_seed") is not None:
        g = np.random.default_rng(spec["bias_seed"])
        bias = (g.standard_normal((spec["bias_rows"], spec["vocab"])) * spec["bias_scale"]).astype(np.float32)
    return ox.LogitsLM(spec["vocab"], ox.hashed_logits_fn(spec["vocab"], spec["seed"], spec["scale"], bias))


def test_logit_trees_match_reference():
    for rec in load("logit_trees.json"):
        if rec["vocab"] > 4096:
            continue  # the V=32000 case runs in the slow tier below
        lm = logits_lm(rec["spec"])
        warp = ox.SamplingConfig(*rec["warp"]) if rec["warp"] else None
        tree = ox.build_sssp(tuple(rec["prefix"]), lm, ox.BuilderParams(rec["K"], rec["D"], rec["B"]), warp)
        assert_tree_matches(tree, rec["tree"], {k: rec[k] for k in ("vocab", "K", "D", "B", "warp")})


@pytest.mark.slow
def test_logit_tree_v32000_matches_reference():
    for rec in load("logit_trees.json"):
        if rec["vocab"] <= 4096:
            continue
        lm = logits_lm(rec["spec"])
        tree = ox.build_sssp(tuple(rec["prefix"]), lm, ox.BuilderParams(rec["K"], rec["D"], rec["B"]), None)
        assert_tree_matches(tree, rec["tree"], rec["vocab"])


def test_logit_engine_matches_reference():
    for rec in load("logit_engine.json"):
        draft, target = logits_lm(rec["draft"]), logits_lm(rec["target"])
        for run in rec["runs"]:
            cfg = ox.SamplingConfig(0.0, 1.0, seed=load("logit_engine.json").index(rec), max_new_tokens=24)
            got, stats = ox.generate_specexec(tuple(rec["prompt"]), draft, target, ox.BuilderParams(rec["K"], rec["D"], rec["B"]), cfg,
                                              warp_scores=(run["scoring"] == "warped"))
            assert got == run["tokens"] == run["sequential"]
            assert stats.target_calls == run["target_calls"] and stats.draft_calls == run["draft_calls"]
            assert stats.accepted_per_iteration == run["accepted"]


def test_specinfer_grid_matches_reference():
    """SpecInfer baseline (specinfer.py:53-127): the oracle's stochastic trees
    (topology, edge log-probs, multiplicities) and full generate_specinfer runs
    equal the reference's on Markov and V=32000 logits pairs."""
    for i, rec in enumerate(load("specinfer_grid.json")):
        if rec["kind"] == "markov":
            target = ox.make_synthetic(rec["target_seed"], rec["V"], rec["sharpness"])
            draft = target.power_smoothed(rec["draft_power"])
        else:
            draft, target = logits_lm(rec["draft"]), logits_lm(rec["target"])
        cfg = ox.SamplingConfig(rec["t"], rec["top_p"], seed=rec["seed"], max_new_tokens=len(rec["tokens"]))
        prompt = tuple(rec["prompt"])
        if "tree" in rec:
            tree = ox.build_stochastic(prompt, draft, rec["branching"], ox.CounterRng(rec["seed"], ox.SI_DRAFT_STREAM), cfg)
            assert [n.parent for n in tree.nodes] == rec["tree"]["parent"], i
            assert [n.token for n in tree.nodes] == rec["tree"]["token"], i
            assert [n.multiplicity for n in tree.nodes] == rec["mult"], i
            for a, b in zip([n.edge_logprob for n in tree.nodes], rec["tree"]["edge"]):
                assert a == b or abs(a - b) <= 1e-12 * max(1.0, abs(b)), i
        toks, st = ox.generate_specinfer(prompt, draft, target, rec["branching"], cfg)
        assert toks == rec["tokens"], i
        assert st.accepted_per_iteration == rec["accepted"] and st.draft_calls == rec["draft_calls"], i


def test_specinfer_schedules():
    assert ox.branching_for_budget(12, 4) == [3, 1, 1, 1]
    assert ox.schedule_size([3, 1, 1, 1]) == 12
    assert ox.branching_for_budget(5, 8) == [1, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        ox.branching_for_budget(0, 3)


def test_beam_instances_match_reference():
    """build_beam (tree.py:330-380): the oracle's trees equal the reference's."""
    for i, rec in enumerate(load("beam_instances.json")):
        if rec["kind"] == "markov":
            model = ox.make_synthetic(rec["seed"], rec["V"], rec["sharpness"])
        else:
            model = logits_lm(rec["spec"])
        warp = ox.SamplingConfig(*rec["warp"]) if rec["warp"] else None
        tree = ox.build_beam(tuple(rec["prompt"]), model, rec["beam"], rec["max_len"], warp)
        assert_tree_matches(tree, rec["tree"], i)
