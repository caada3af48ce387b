"""SpecInfer baseline on the GPU: stochastic trees and
generate_specinfer runs vs the reference fixtures and the CPU oracle (bit-exact
trees: parents, tokens, float64 edge log-probs, multiplicities), Llama-shaped
runs vs the oracle replayed on the GPU's own rows, and t=0 == greedy decoding."""

import json
import pathlib

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import speckit_oracle as ox
from paper_2406_02532_b200 import specinfer as si
from paper_2406_02532_b200.llama import LlamaModel, SyntheticBias

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())["data"]


def test_markov_specinfer_matches_reference_and_oracle(cuda):
    n = 0
    for i, rec in enumerate(load("specinfer_grid.json")):
        if rec["kind"] != "markov":
            continue
        n += 1
        tg = sx.make_synthetic(rec["target_seed"], rec["V"], rec["sharpness"])
        dg = tg.power_smoothed(rec["draft_power"])
        to = ox.make_synthetic(rec["target_seed"], rec["V"], rec["sharpness"])
        do = to.power_smoothed(rec["draft_power"])
        prompt, br = tuple(rec["prompt"]), rec["branching"]
        cfg = sx.SamplingConfig(rec["t"], rec["top_p"], seed=rec["seed"], max_new_tokens=len(rec["tokens"]))
        ocfg = ox.SamplingConfig(rec["t"], rec["top_p"], seed=rec["seed"], max_new_tokens=len(rec["tokens"]))
        g = si.build_stochastic(prompt, dg, br, sx.CounterRng(rec["seed"], si.DRAFT_STREAM), cfg)
        o = ox.build_stochastic(prompt, do, br, ox.CounterRng(rec["seed"], ox.SI_DRAFT_STREAM), ocfg)
        assert [(x.parent, x.token, x.multiplicity) for x in g.nodes] == \
            [(x.parent, x.token, x.multiplicity) for x in o.nodes], i
        assert [x.edge_logprob for x in g.nodes] == [x.edge_logprob for x in o.nodes], i
        assert g.rounds == o.rounds
        assert [x.parent for x in g.nodes] == rec["tree"]["parent"] and [x.multiplicity for x in g.nodes] == rec["mult"]
        for nid in list(o.draft_dists):
            assert np.array_equal(g.draft_dists[nid], o.draft_dists[nid]), (i, nid)
        toks, st = sx.generate_specinfer(prompt, dg, tg, br, cfg)
        assert toks == rec["tokens"], i
        assert st.accepted_per_iteration == rec["accepted"] and st.draft_calls == rec["draft_calls"], i
    assert n >= 50


def test_verify_matches_oracle_rng_consumption(cuda):
    """The device walk consumes exactly the uniforms the oracle consumes."""
    tg, to = sx.make_synthetic(11, 9, 0.4), ox.make_synthetic(11, 9, 0.4)
    dg, do = tg.power_smoothed(0.5), to.power_smoothed(0.5)
    for seed in range(20):
        cfg = sx.SamplingConfig(0.8, 0.95, seed=seed)
        g = si.build_stochastic((1, 2), dg, [4, 2, 2], sx.CounterRng(seed, "d"), cfg)
        o = ox.build_stochastic((1, 2), do, [4, 2, 2], ox.CounterRng(seed, "d"), ox.SamplingConfig(0.8, 0.95, seed=seed))
        rg, ro = sx.CounterRng(seed, "a"), ox.CounterRng(seed, "a")
        vg = si.verify_specinfer(g, tg, cfg, rg)
        vo = ox.verify_specinfer(o, to, ox.SamplingConfig(0.8, 0.95, seed=seed), ro)
        assert (vg.accepted_path, vg.bonus_token) == (vo.accepted_path, vo.bonus_token)
        assert rg.counter == ro.counter


def test_contract_errors(cuda):
    m = sx.make_synthetic(1, 5, 0.5)
    tree = sx.build_sssp((0,), m, sx.BuilderParams(4, 2, 2))
    with pytest.raises(ValueError):
        si.verify_specinfer(tree, m, sx.SamplingConfig(1.0, 1.0), sx.CounterRng(0, "a"))
    with pytest.raises(ValueError):
        si.build_stochastic((0,), m, [], sx.CounterRng(0, "d"))
    with pytest.raises(ValueError):
        si.build_stochastic((0,), m, [2, 0], sx.CounterRng(0, "d"))


@pytest.fixture(scope="module")
def llama_pair():
    torch.cuda.set_device(0)
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    target = LlamaModel("tiny", seed=1, max_ctx=4096, max_tokens=512, synthetic=syn)
    draft = LlamaModel("tiny-draft", seed=2, max_ctx=4096, max_tokens=512, synthetic=syn)
    return draft, target


@pytest.mark.parametrize("t,p", [(0.6, 0.9), (1.0, 1.0), (0.8, 0.95)])
def test_llama_specinfer_replay_parity(llama_pair, monkeypatch, t, p):
    draft, target = llama_pair
    draft.record, target.record = [], []
    prompt = tuple(int(x) for x in np.random.default_rng(3).integers(0, 32000, size=20))
    br = si.branching_for_budget(24, 4)
    got, st = sx.generate_specinfer(prompt, draft, target, br, sx.SamplingConfig(t, p, seed=5, max_new_tokens=30))
    drec, trec = draft.record, target.record
    draft.record = target.record = None
    state = {"k": -1}

    def lm(recs):
        return ox.LogitsLM(32000, lambda ps: np.stack([recs[state["k"]][tuple(q)] for q in ps]))

    real = ox.build_stochastic

    def bs(*a, **kw):
        state["k"] += 1
        return real(*a, **kw)

    monkeypatch.setattr(ox, "build_stochastic", bs)
    exp, ost = ox.generate_specinfer(prompt, lm(drec), lm(trec), br, ox.SamplingConfig(t, p, seed=5, max_new_tokens=30))
    assert got == exp
    assert st.accepted_per_iteration == ost.accepted_per_iteration and st.draft_calls == ost.draft_calls
    assert st.generation_rate > 1.0


def test_llama_specinfer_greedy_equals_sequential(llama_pair):
    draft, target = llama_pair
    prompt = tuple(range(900, 916))
    cfg = sx.SamplingConfig(0.0, 1.0, seed=0, max_new_tokens=24)
    got, _ = sx.generate_specinfer(prompt, draft, target, si.branching_for_budget(16, 4), cfg)
    seq, _ = sx.generate_sequential(prompt, target, cfg)
    assert got == seq
