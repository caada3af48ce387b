"""Tensor-parallel target on the GPU (tp.py, llama.py): the sharded kernels
(local heads / FFN slice / vocab slice, all-reduced o and down projections,
all-gathered logits) reproduce the unsharded model, and a SpecExec run with a
TP target gives bit-identical tokens on every rank, equal to the CPU oracle
replayed on the GPU's own rows. Ranks run as threads sharing cuda:0
(ThreadComm) -- the same model code as NCCL ranks on separate GPUs."""

import threading

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import llama_ref
from oracle import speckit_oracle as ox
from paper_2406_02532_b200.llama import LlamaConfig, LlamaModel, SyntheticBias
from paper_2406_02532_b200.tp import ThreadComm

pytestmark = pytest.mark.gpu
CFG = LlamaConfig(32000, 256, 2, 4, 2, 512, 1e4, 1e-5, name="tiny-tp")


def run_ranks(world, fn):
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("world", [2])
def test_tp_logits_match_unsharded(cuda, world, fused):
    full = LlamaModel(CFG, seed=3, max_ctx=1024, max_tokens=256)
    prefix = tuple(int(t) for t in np.random.default_rng(1).integers(0, 32000, size=40))
    exp = full.prefix_rows(prefix)[0].clone()
    W = full.w.to_cpu_fp32()
    cpu = llama_ref.forward_logits(CFG, W, list(prefix))[-1]
    assert (exp.cpu() - cpu).abs().max().item() < 2e-2
    for reduce_bf16, tol in ((False, 1e-2), (True, 2e-2)):
        comms = ThreadComm.group(world)
        outs = run_ranks(world, lambda r: LlamaModel(CFG, seed=3, max_ctx=1024, max_tokens=256, tp=comms[r],
                                                     reduce_bf16=reduce_bf16, tp_fused=fused)
                         .prefix_rows(prefix)[0].clone())
        for o in outs[1:]:
            assert torch.equal(o, outs[0])  # every rank holds identical all-gathered rows
        assert (outs[0] - exp).abs().max().item() < tol, reduce_bf16
        assert (outs[0].cpu() - cpu).abs().max().item() < 2e-2


@pytest.mark.parametrize("fused", [False, True])
def test_tp_target_generation_ranks_agree_replay_parity(cuda, monkeypatch, fused):
    world = 2
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    comms = ThreadComm.group(world)
    prompt = tuple(int(x) for x in np.random.default_rng(9).integers(0, 32000, size=24))
    params = sx.BuilderParams(64, 8, 16)
    cfg = sx.SamplingConfig(0.0, 1.0, seed=3, max_new_tokens=40)

    def rank(r):
        target = LlamaModel(CFG, seed=3, max_ctx=2048, max_tokens=512, synthetic=syn, tp=comms[r], tp_fused=fused)
        draft = LlamaModel("tiny-draft", seed=2, max_ctx=4096, max_tokens=512, synthetic=syn)
        draft.use_graphs = False  # no concurrent graph capture from two threads
        if r == 0:
            draft.record, target.record = [], []
        toks, st = sx.generate_specexec(prompt, draft, target, params, cfg, warp_scores=False)
        return toks, st, draft.record, target.record

    outs = run_ranks(world, rank)
    toks, st, drec, trec = outs[0]
    for o in outs[1:]:
        assert o[0] == toks and o[1].accepted_per_iteration == st.accepted_per_iteration
    assert st.generation_rate > 1.0
    # the oracle rebuilds every tree and walk from rank 0's recorded rows
    state = {"k": -1}

    def lm(recs):
        return ox.LogitsLM(32000, lambda ps: np.stack([recs[state["k"]][tuple(p)] for p in ps]))

    real = ox.precompute

    def pre(prefix, d, t, prm, warp=None, warp_scores=True):
        state["k"] += 1
        return real(prefix, d, t, prm, warp, warp_scores)

    monkeypatch.setattr(ox, "precompute", pre)
    exp, ost = ox.generate_specexec(prompt, lm(drec), lm(trec), ox.BuilderParams(64, 8, 16),
                                    ox.SamplingConfig(0.0, 1.0, seed=3, max_new_tokens=40), warp_scores=False)
    assert toks == exp and st.accepted_per_iteration == ost.accepted_per_iteration


def test_tp_argmax_keys_walk_equals_gathered_rows(cuda):
    """KV1: with tp_argmax the TP target returns one int64 argmax key per tree
    row (a MAX all-reduce over the vocab slices) instead of all-gathered logits;
    the t = 0 SpecExec run is token-for-token the gathered-rows run on every rank,
    a t > 0 walk is refused, and a full-row read raises."""
    world = 2
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    prompt = tuple(int(x) for x in np.random.default_rng(11).integers(0, 32000, size=24))
    params = sx.BuilderParams(64, 8, 16)
    cfg = sx.SamplingConfig(0.0, 1.0, seed=3, max_new_tokens=40)
    res = {}
    for argmax in (False, True):
        comms = ThreadComm.group(world)

        def rank(r):
            target = LlamaModel(CFG, seed=3, max_ctx=2048, max_tokens=512, synthetic=syn, tp=comms[r],
                                tp_fused=False, tp_argmax=argmax)
            draft = LlamaModel("tiny-draft", seed=2, max_ctx=4096, max_tokens=512, synthetic=syn)
            draft.use_graphs = False
            toks, st = sx.generate_specexec(prompt, draft, target, params, cfg, warp_scores=False)
            extra = None
            if argmax:
                cache = sx.precompute(prompt + tuple(toks), draft, target, params, cfg, warp_scores=False)
                assert cache.dists.rows.dtype == torch.int64
                with pytest.raises(RuntimeError):
                    cache.current_dist()
                with pytest.raises(ValueError):
                    cache.walk(np.zeros(4), sx.SamplingConfig(0.6, 0.9, seed=0), 4)
                extra = True
            return toks, st.accepted_per_iteration, extra

        res[argmax] = run_ranks(world, rank)
    for r in range(world):
        assert res[True][r][0] == res[False][r][0] == res[False][0][0]
        assert res[True][r][1] == res[False][r][1]


def test_rows_argmax_packed_kernel(cuda):
    """sx_rows_argmax_packed on vocab slices, max-combined: the global argmax with
    the lowest id on exact ties (np.argmax), for negative / positive logits."""
    from paper_2406_02532_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(5)
    n, V, W = 37, 1000, 4
    z = torch.randn(n, V, device="cuda", generator=g) * 3
    z[3, 10] = z[3, 700] = z[3].max() + 1.0  # exact tie across slices -> lowest id
    z[4, :] = -2.5  # all equal -> id 0
    z[5, 999] = 1e30
    keys = torch.zeros(W, n, 1, dtype=torch.int64, device="cuda")
    Vl = V // W
    for w in range(W):
        K.rows_argmax_packed(z[:, w * Vl:(w + 1) * Vl], w * Vl, keys[w])
    best = keys.max(0).values[:, 0]
    got = (0x7FFFFFFF - (best & 0x7FFFFFFF)).cpu().numpy()
    exp = np.argmax(z.cpu().numpy(), axis=1)
    assert (got == exp).all()
    assert got[3] == 10 and got[4] == 0 and got[5] == 999
