"""Stage-1 A/B knobs build the same tree: every env-selected variant of the
chunked logits-row path and of the update kernel (the earlier implementation
each round-2 change replaced) must give the default's tree node for node, on
the same draft rows (a Llama-shaped draft with a low-rank logit bias, so the
rounds have survivors and both update paths run). Each variant runs in its own
process: the knobs are read once per process."""

import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]

CHILD = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2406_02532_b200 as sx
from paper_2406_02532_b200.llama import LlamaConfig, LlamaModel, SyntheticBias
V, K, D, B = 32000, 2048, 10, 256
cfg = LlamaConfig(V, 256, 2, 2, 1, 512, 1e4, 1e-5, name="variants")
draft = LlamaModel(cfg, seed=13, max_ctx=4 * K + 2 * B * (D + 1) + 256, max_tokens=B,
                   synthetic=SyntheticBias(seed=5, rank=64, scale=3.0))
prompt = tuple(int(t) for t in np.random.default_rng(77).integers(0, V, size=12))
out = []
for warp in (None, sx.SamplingConfig(0.6, 0.9, seed=0)):
    draft.committed.clear()
    g = sx.build_sssp(prompt, draft, sx.BuilderParams(K, D, B), warp, warp_scores=warp is not None)
    key = [(n.parent, n.token, n.edge_logprob.hex()) for n in g.nodes]
    out.append([hashlib.sha256(json.dumps(key).encode()).hexdigest(), g.rounds, len(g.nodes)])
print(json.dumps(out))
"""

VARIANTS = [{}, {"SX_TREE_MERGE": "0"}, {"SX_TREE_FUSED_EXACT": "0"}, {"SX_TREE_PDL": "0"},
            {"SX_TREE_SORT_REG": "0"}, {"SX_TREE_MAX_PIPE": "0"}, {"SX_TREE_MAX_PIPE": "2"}]


def _build(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_stage1_variants_build_the_same_tree(cuda):
    ref = _build(VARIANTS[0])
    assert ref[0][2] == 2048 and ref[0][1] > 2
    for v in VARIANTS[1:]:
        assert _build(v) == ref, v
