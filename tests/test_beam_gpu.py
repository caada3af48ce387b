"""build_beam on the GPU (tree.py:330-380): trees equal the
reference fixtures (topology, rounds, edges within the oracle's 1e-12) and the
CPU oracle bit for bit; Llama-shaped draft vs the oracle replayed on the GPU's
own rows; beam 1 is the greedy chain."""

import json
import pathlib

import numpy as np
import pytest

import paper_2406_02532_b200 as sx
from oracle import speckit_oracle as ox
from paper_2406_02532_b200.llama import LlamaModel, SyntheticBias

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())["data"]


def test_beam_markov_vs_reference_and_oracle(cuda):
    n = 0
    for i, rec in enumerate(load("beam_instances.json")):
        if rec["kind"] != "markov":
            continue
        n += 1
        g_model = sx.make_synthetic(rec["seed"], rec["V"], rec["sharpness"])
        o_model = ox.make_synthetic(rec["seed"], rec["V"], rec["sharpness"])
        gw = sx.SamplingConfig(*rec["warp"]) if rec["warp"] else None
        ow = ox.SamplingConfig(*rec["warp"]) if rec["warp"] else None
        g = sx.build_beam(tuple(rec["prompt"]), g_model, rec["beam"], rec["max_len"], gw)
        o = ox.build_beam(tuple(rec["prompt"]), o_model, rec["beam"], rec["max_len"], ow)
        assert [(x.parent, x.token, x.edge_logprob) for x in g.nodes] == \
            [(x.parent, x.token, x.edge_logprob) for x in o.nodes], i
        assert g.rounds == o.rounds == rec["tree"]["rounds"], i
        assert [x.parent for x in g.nodes] == rec["tree"]["parent"], i
        assert [x.token for x in g.nodes] == rec["tree"]["token"], i
    assert n >= 70


def test_beam_one_is_greedy_chain(cuda):
    chain = sx.MarkovModel(np.roll(np.eye(4), 1, axis=1) * 0.7 + 0.075, order=1)
    tree = sx.build_beam((0,), chain, 1, 4)
    assert [n.token for n in tree.nodes] == [1, 2, 3, 0]
    assert [n.parent for n in tree.nodes] == [-1, 0, 1, 2]
    with pytest.raises(ValueError):
        sx.build_beam((0,), chain, 0, 3)


@pytest.mark.parametrize("warp", [None, (0.6, 0.9)])
def test_beam_llama_replay(cuda, warp):
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    draft = LlamaModel("tiny-draft", seed=2, max_ctx=2048, max_tokens=256, synthetic=syn)
    draft.record = []
    prompt = tuple(int(x) for x in np.random.default_rng(11).integers(0, 32000, size=12))
    g = sx.build_beam(prompt, draft, 16, 5, sx.SamplingConfig(*warp) if warp else None)
    tab = draft.record[-1]
    draft.record = None
    lm = ox.LogitsLM(32000, lambda ps: np.stack([tab[tuple(q)] for q in ps]))
    o = ox.build_beam(prompt, lm, 16, 5, ox.SamplingConfig(*warp) if warp else None)
    assert [(x.parent, x.token, x.edge_logprob) for x in g.nodes] == \
        [(x.parent, x.token, x.edge_logprob) for x in o.nodes]
    assert g.rounds == o.rounds and len(g.nodes) >= 16
