"""Logit parity at the named architectures (SURVEY 8(d) shapes at real width):
2-layer truncations of Llama-2-7B / Llama-2-70B / Llama-3-8B / Llama-3-70B
(the first two decoder layers of the seeded full models -- same draw order),
bf16 weights, against the fp32 CPU oracle (oracle/llama_ref.py) on the same
weights, within the north_star bf16 tolerance 2e-2 abs:

* prefill rows (causal chain through the prefix cache) of draft and target;
* every draft row of a K=1024, B=1024 GPU tree build (the batched tree rounds
  with ancestor-slot attention over the draft KV);
* every row of the target's ONE pass over anchor + 1024 tree nodes (tree-masked
  attention, fused QKV+RoPE epilogue, GQA 64/8, ff 28672 / 14336, V 32000 / 128256,
  theta 1e4 / 5e5).

The CPU side is `forward_tree_logits` -- the flattened ancestor mask of
pkg/src/speckit/tree.py:208-219, pinned to full-prefix forwards by
tests/test_llama_ref_cpu.py."""

import dataclasses
import gc

import numpy as np
import pytest
import torch

import paper_2406_02532_b200 as sx
from oracle import llama_ref
from paper_2406_02532_b200.llama import PRESETS, LlamaModel

pytestmark = pytest.mark.gpu
TOL = 2e-2
PAIRS = [("llama2-7b", "llama2-70b"), ("llama3-8b", "llama3-70b")]
K, D, B, P = 1024, 16, 1024, 128


def truncated(name: str, layers: int = 2):
    return dataclasses.replace(PRESETS[name], layers=layers, name=f"{name}-L{layers}")


@pytest.fixture(scope="module", params=PAIRS, ids=["llama2", "llama3"])
def named_pair(request):
    torch.cuda.set_device(0)
    dname, tname = request.param
    draft = LlamaModel(truncated(dname), seed=2, max_ctx=P + 4 * K + 2 * B * (D + 1) + 64, max_tokens=B + 1)
    target = LlamaModel(truncated(tname), seed=1, max_ctx=P + K + 64, max_tokens=K + 1)
    yield draft, target
    del draft, target
    gc.collect()
    torch.cuda.empty_cache()


def _prompt(V, seed=0):
    return [int(t) for t in np.random.default_rng(seed).integers(0, V, size=P)]


def _max_err(got: torch.Tensor, exp: torch.Tensor) -> float:
    return float((got.float().cpu() - exp).abs().max())


def test_prefill_rows(named_pair):
    for m in named_pair:
        prompt = _prompt(m.cfg.vocab, 11)
        W = m.w.to_cpu_fp32()
        exp = llama_ref.forward_logits(m.cfg, W, prompt)
        for n in (1, 37, P):
            got = m.prefix_rows(prompt[:n])[0]
            err = _max_err(got, exp[n - 1])
            assert err < TOL, (m.cfg.name, n, err)


def test_tree_build_and_target_pass_rows(named_pair):
    draft, target = named_pair
    prompt = _prompt(target.cfg.vocab, 5)
    draft.record = []
    try:
        tree = sx.build_sssp(tuple(prompt), draft, sx.BuilderParams(K, D, B), None, warp_scores=False)
        rec = draft.record[-1]
    finally:
        draft.record = None
    assert len(tree.nodes) == K
    # every draft row the builder consumed (root + each expanded node)
    paths = sorted((k[P:] for k in rec if len(k) > P), key=len)
    exp_d = llama_ref.forward_tree_logits(draft.cfg, draft.w.to_cpu_fp32(), prompt, paths)
    got_d = torch.stack([torch.from_numpy(rec[tuple(prompt)])] + [torch.from_numpy(rec[tuple(prompt) + p]) for p in paths])
    err_d = _max_err(got_d, exp_d)
    assert err_d < TOL, ("draft rows", len(paths), err_d)
    # the target's one pass over anchor + every node
    rows = target.tree_rows(tree)
    assert rows.shape == (K + 1, target.cfg.vocab)
    tpaths = [tree.path_tokens(i) for i in range(K)]
    exp_t = llama_ref.forward_tree_logits(target.cfg, target.w.to_cpu_fp32(), prompt, tpaths)
    err_t = _max_err(rows, exp_t)
    assert err_t < TOL, ("target rows", err_t)
