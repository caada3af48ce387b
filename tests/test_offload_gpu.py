"""Stage 3 anchored to the oracle: the offloaded target (weights in pinned host
RAM, streamed per layer through the HBM ring by LayerStreamer / sx_stream_copy)
against the fp32 CPU forward (oracle/llama_ref.py) -- not only against the
resident GPU path:

* tiny (d=256): prefill rows and every tree-pass row within 2e-2 abs;
* a 2-layer Llama-2-70B-width target streamed through a 2-slot ring: tree-pass
  rows no further from the fp32 forward than the bf16 policy itself
  (tests/test_named_configs_gpu.check);
* tokens: SpecExec with the offloaded target at t=0.6 / top-p 0.9 (the C3
  sampling) replays bit-exactly through the oracle engine on the recorded rows,
  and equals sequential decoding at t=0."""

import dataclasses

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import llama_ref
from oracle import speckit_oracle as ox
from paper_2406_02532_b200.llama import PRESETS, LlamaModel, SyntheticBias

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _bias(m):
    return (m.bias_u.float().cpu(), m.bias_w.float().cpu()) if m.synthetic is not None else None


def test_offloaded_tiny_vs_fp32_oracle(cuda):
    syn = SyntheticBias(seed=7, rank=64, scale=4.0)
    tgt = LlamaModel("tiny", seed=3, max_ctx=2048, max_tokens=512, synthetic=syn, offload=True, offload_buffers=3)
    drf = LlamaModel("tiny-draft", seed=4, max_ctx=4096, max_tokens=512, synthetic=syn)
    W = tgt.w.to_cpu_fp32()
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 32000, size=40)]
    exp = llama_ref.forward_logits(tgt.cfg, W, prompt, _bias(tgt))
    for n in (1, 17, 40):
        assert float((tgt.prefix_rows(prompt[:n])[0].cpu() - exp[n - 1]).abs().max()) < TOL
    tree = sx.build_sssp(tuple(prompt), drf, sx.BuilderParams(200, 8, 32), None, warp_scores=False)
    rows = tgt.tree_rows(tree).cpu()
    paths = [tree.path_tokens(i) for i in range(len(tree.nodes))]
    exp_t = llama_ref.forward_tree_logits(tgt.cfg, W, prompt, paths, _bias(tgt))
    assert float((rows - exp_t).abs().max()) < TOL
    assert tgt.streamer.bytes >= tgt.w.layer_bytes * tgt.cfg.layers * 3


def test_offloaded_70b_width_vs_oracle(cuda):
    from test_named_configs_gpu import check

    cfg = dataclasses.replace(PRESETS["llama2-70b"], layers=2, name="llama2-70b-L2")
    dcfg = dataclasses.replace(PRESETS["llama2-7b"], layers=1, name="llama2-7b-L1")
    tgt = LlamaModel(cfg, seed=1, max_ctx=1024, max_tokens=520, offload=True, offload_buffers=2)
    drf = LlamaModel(dcfg, seed=2, max_ctx=4096, max_tokens=128)
    W = tgt.w.to_cpu_fp32()
    prompt = [int(t) for t in np.random.default_rng(9).integers(0, cfg.vocab, size=64)]
    tree = sx.build_sssp(tuple(prompt), drf, sx.BuilderParams(511, 10, 128), None, warp_scores=False)
    rows = tgt.tree_rows(tree)
    paths = [tree.path_tokens(i) for i in range(len(tree.nodes))]
    check(rows, lambda pol: llama_ref.forward_tree_logits(cfg, W, prompt, paths, policy=pol),
          "llama2-70b-L2 offloaded tree pass (512 rows)")


@pytest.mark.parametrize("t,top_p", [(0.6, 0.9), (0.0, 1.0)])
def test_offloaded_specexec_replay_parity(cuda, monkeypatch, t, top_p):
    syn = SyntheticBias(seed=8, rank=64, scale=4.0)
    tgt = LlamaModel("tiny", seed=5, max_ctx=2048, max_tokens=256, synthetic=syn, offload=True, offload_buffers=2)
    drf = LlamaModel("tiny-draft", seed=6, max_ctx=4096, max_tokens=256, synthetic=syn)
    prompt = tuple(int(x) for x in np.random.default_rng(21).integers(0, 32000, size=30))
    params = sx.BuilderParams(96, 8, 16)
    cfg = sx.SamplingConfig(t, top_p, seed=2, max_new_tokens=30)
    drf.record, tgt.record = [], []
    got, st = sx.generate_specexec(prompt, drf, tgt, params, cfg, warp_scores=t > 0)
    d_rec, t_rec = drf.record, tgt.record
    drf.record = tgt.record = None
    state = {"k": -1}
    lm = lambda recs: ox.LogitsLM(32000, lambda ps: np.stack([recs[state["k"]][tuple(q)] for q in ps]))  # noqa: E731
    real = ox.precompute

    def pre(*a, **kw):
        state["k"] += 1
        return real(*a, **kw)

    monkeypatch.setattr(ox, "precompute", pre)
    exp, ost = ox.generate_specexec(prompt, lm(d_rec), lm(t_rec), ox.BuilderParams(96, 8, 16),
                                    ox.SamplingConfig(t, top_p, seed=2, max_new_tokens=30), warp_scores=t > 0)
    assert got == exp and st.accepted_per_iteration == ost.accepted_per_iteration
    if t == 0.0:
        seq, _ = sx.generate_sequential(prompt, tgt, cfg)
        assert got == seq
