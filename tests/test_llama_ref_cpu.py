"""The fp32 CPU logit oracle's tree forward (oracle/llama_ref.forward_tree_logits,
the flattened ancestor mask of pkg/src/speckit/tree.py:208-219) equals the plain
causal forward of every node's full prefix -- the stateless meaning of the
reference's `next_distributions` (pkg/src/speckit/models.py:47-52). CPU only."""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import llama_ref
from paper_2406_02532_b200.llama import PRESETS


def cpu_weights(cfg, seed):
    g = torch.Generator().manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=g) * 0.05  # noqa: E731
    layers = [{"wqkv": r(cfg.qkv_out, cfg.d), "wo": r(cfg.d, cfg.heads * cfg.head_dim), "wg": r(cfg.ff, cfg.d),
               "wu": r(cfg.ff, cfg.d), "wd": r(cfg.d, cfg.ff), "n1": 1 + r(cfg.d), "n2": 1 + r(cfg.d)}
              for _ in range(cfg.layers)]
    return {"emb": r(cfg.vocab, cfg.d), "layers": layers, "nf": 1 + r(cfg.d), "lm": r(cfg.vocab, cfg.d)}


@pytest.mark.parametrize("name,kvh", [("tiny", 1), ("tiny-draft", 2)])
def test_tree_forward_equals_full_prefix_forward(name, kvh):
    cfg = dataclasses.replace(PRESETS[name], vocab=500, kv_heads=kvh)
    W = cpu_weights(cfg, 3)
    rng = np.random.default_rng(1)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, size=9)]
    paths: list[tuple[int, ...]] = []
    for _ in range(40):  # random prefix-closed tree, parents first, siblings distinct
        par = paths[int(rng.integers(0, len(paths)))] if paths and rng.random() < 0.8 else ()
        if len(par) >= 6:
            continue
        tok = int(rng.integers(0, cfg.vocab))
        if par + (tok,) not in paths:
            paths.append(par + (tok,))
    rows = llama_ref.forward_tree_logits(cfg, W, prompt, paths)
    assert rows.shape == (len(paths) + 1, cfg.vocab)
    torch.testing.assert_close(rows[0], llama_ref.forward_logits(cfg, W, prompt)[-1], atol=1e-3, rtol=1e-3)
    for i, path in enumerate(paths):
        exp = llama_ref.forward_logits(cfg, W, prompt + list(path))[-1]
        torch.testing.assert_close(rows[i + 1], exp, atol=1e-3, rtol=1e-3)  # mask semantics: a wrong key set is O(1)


def test_tree_forward_rejects_unclosed_paths():
    cfg = dataclasses.replace(PRESETS["tiny"], vocab=50)
    W = cpu_weights(cfg, 0)
    with pytest.raises(ValueError):
        llama_ref.forward_tree_logits(cfg, W, [1, 2], [(3, 4)])


def test_cpu_llama_lm_rows_equal_stateless_forwards():
    """CpuLlamaLM (the timed CPU reference path) batches a draft round / target
    pass as one tree forward; each row must equal its own causal forward."""
    cfg = dataclasses.replace(PRESETS["tiny"], vocab=300)
    W = cpu_weights(cfg, 5)
    lm = llama_ref.CpuLlamaLM(cfg, W)
    prompt = (4, 8, 15, 16)
    batch = [prompt, prompt + (23,), prompt + (23, 42), prompt + (7, 1, 2), prompt + (9,)]
    rows = lm.logits(batch)
    for p, r in zip(batch, rows):
        torch.testing.assert_close(r, llama_ref.forward_logits(cfg, W, list(p))[-1], atol=1e-3, rtol=1e-3)
    # unrelated prefixes (no shared first token) fall back to one forward each
    rows = lm.logits([(1, 2), (3,)])
    torch.testing.assert_close(rows[1], llama_ref.forward_logits(cfg, W, [3])[-1], atol=1e-3, rtol=1e-3)
    d = lm.next_distributions(batch[:2])
    assert d.shape == (2, cfg.vocab) and abs(d.sum(axis=1) - 1).max() < 1e-12


def test_host_weight_draw_matches_device_layout_shapes():
    from paper_2406_02532_b200.llama import host_weights_fp32

    cfg = PRESETS["tiny-draft"]
    a, b = host_weights_fp32(cfg, 3), host_weights_fp32(cfg, 3)
    assert torch.equal(a["lm"], b["lm"]) and a["layers"][1]["wd"].shape == (cfg.d, cfg.ff)
    assert torch.equal(a["emb"], a["emb"].bfloat16().float())  # bf16 values
