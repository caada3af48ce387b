"""Full-size C2 replay parity (BASELINE configs[1]): the real Llama-2-7B-shaped
draft and Llama-2-70B-shaped target (random-init bf16, target resident in HBM),
K=1024, D=16, B=1024 -- the bench workload. Each GPU iteration's draft rows and
target rows are recorded (fp32 logits), then the CPU oracle
(oracle/speckit_oracle.py: build_sssp tree.py:240-327, precompute
engine.py:73-89, generate_specexec engine.py:92-131) is run on those same rows
(the ReplayLM construction of SURVEY 8(c)). The trees (ids, parents, tokens,
edge log-probs, rounds), the accepted tokens and GenStats must be identical:

* t=0, raw draft scoring (the bench headline);
* t=0.6 / top-p 0.9 with warped scoring (the C3 sampling configuration)."""

import gc

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import speckit_oracle as ox
from paper_2406_02532_b200 import engine as E
from paper_2406_02532_b200.llama import LlamaModel

pytestmark = pytest.mark.gpu
K, D, B, P = 1024, 16, 1024, 128


@pytest.fixture(scope="module")
def c2_pair():
    torch.cuda.set_device(0)
    gc.collect()
    torch.cuda.empty_cache()
    target = LlamaModel("llama2-70b", seed=1, max_ctx=P + 8 * (D + 1) + K + 64, max_tokens=K + 1)
    draft = LlamaModel("llama2-7b", seed=2, max_ctx=P + 8 * (D + 1) + 4 * K + 2 * B * (D + 1) + 64, max_tokens=B)
    yield draft, target
    del draft, target
    gc.collect()
    torch.cuda.empty_cache()


def _nodes(tree):
    return [(n.parent, n.token, n.edge_logprob, n.cum_logprob) for n in tree.nodes]


@pytest.mark.parametrize("t,top_p,warp_scores,new", [(0.0, 1.0, False, 3), (0.6, 0.9, True, 3)],
                         ids=["t0-raw", "t0.6-p0.9-warped"])
def test_c2_iterations_replay_bit_exact(c2_pair, monkeypatch, t, top_p, warp_scores, new):
    draft, target = c2_pair
    V = target.cfg.vocab
    prompt = tuple(int(x) for x in np.random.default_rng(1000 + int(t * 10)).integers(0, V, size=P))
    cfg = sx.SamplingConfig(t, top_p, seed=0, max_new_tokens=new)
    gpu_trees = []
    real_pre = E.precompute

    def rec_pre(*a, **kw):
        cache = real_pre(*a, **kw)
        gpu_trees.append(cache.tree)
        return cache

    monkeypatch.setattr(E, "precompute", rec_pre)
    draft.record, target.record = [], []
    try:
        got, stats = sx.generate_specexec(prompt, draft, target, sx.BuilderParams(K, D, B), cfg, warp_scores=warp_scores)
        d_rec, t_rec = draft.record, target.record
    finally:
        draft.record = target.record = None
    monkeypatch.setattr(E, "precompute", real_pre)
    assert len(got) == new and len(gpu_trees) == stats.target_calls == len(t_rec)
    assert all(len(tr.nodes) == K for tr in gpu_trees)

    state = {"k": -1}
    ox_trees = []

    def lm(recs):
        return ox.LogitsLM(V, lambda ps: np.stack([recs[state["k"]][tuple(p)] for p in ps]))

    real_ox = ox.precompute

    def ox_pre(prefix, d, tg, params, warp=None, ws=True):
        state["k"] += 1
        cache = real_ox(prefix, d, tg, params, warp, ws)
        ox_trees.append(cache.tree)
        return cache

    monkeypatch.setattr(ox, "precompute", ox_pre)
    exp, ostats = ox.generate_specexec(prompt, lm(d_rec), lm(t_rec), ox.BuilderParams(K, D, B),
                                       ox.SamplingConfig(t, top_p, seed=0, max_new_tokens=new), warp_scores=warp_scores)
    assert got == exp
    assert stats.accepted_per_iteration == ostats.accepted_per_iteration
    assert stats.draft_calls == ostats.draft_calls and stats.target_calls == ostats.target_calls
    assert len(ox_trees) == len(gpu_trees)
    for g, o in zip(gpu_trees, ox_trees):
        assert _nodes(g) == _nodes(o)
        assert g.rounds == o.rounds
