"""SpecInfer baseline on the GPU: stochastic drafting + multi-round rejection
verification (the paper's SX-vs-SI comparison).

API of the reference (pkg/src/speckit/specinfer.py): `DRAFT_STREAM` /
`ACCEPT_STREAM` (:26-27), `VerifyOutcome` (:30-39), `verify_specinfer`
(:53-96), `generate_specinfer` (:99-127), `branching_for_budget` (:130-143),
`schedule_size` (:146-153); and `build_stochastic` (tree.py:383-425).

Device path per iteration: each level of the stochastic tree is ONE draft
forward over the level's nodes (rows stay on the GPU), the canonical warp of
those rows (sx_warp_rows) and all `width` i.i.d. draws per node in one launch
(sx_sample_rows_idx, uniforms of the host CounterRng "specinfer-draft"
stream); duplicate draws merge on the host (multiplicity). Verification is one
target pass over the anchor + every node and one CTA walking the tree
(sx_specinfer_verify) with the "specinfer-accept" uniforms. The sampled-from
distributions q never leave the device; `tree.draft_dists` maps node -> row.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .engine import GenStats
from .models import as_device_model
from .rng import CounterRng
from .sampling import SamplingConfig
from .tree import ROOT, DraftTree

DRAFT_STREAM = "specinfer-draft"
ACCEPT_STREAM = "specinfer-accept"


@dataclass
class VerifyOutcome:
    """Result of verifying one draft tree (specinfer.py:30-39)."""

    accepted_path: list[int]
    bonus_token: int

    @property
    def tokens_emitted(self) -> int:
        return len(self.accepted_path) + 1


class DeviceDists:
    """tree.draft_dists on the device: node id (ROOT = -1) -> row of `rows`
    (fp64 [*, V]); indexing materialises the float64 row on the host."""

    def __init__(self, rows: torch.Tensor):
        self.rows = rows
        self.row_of: dict[int, int] = {}

    def __contains__(self, node: int) -> bool:
        return node in self.row_of

    def __getitem__(self, node: int) -> np.ndarray:
        return self.rows[self.row_of[node]].cpu().numpy()

    def __len__(self) -> int:
        return len(self.row_of)


def _check_schedule(branching) -> list[int]:
    if not branching:
        raise ValueError("branching schedule must be non-empty")
    if any(int(w) < 1 for w in branching):
        raise ValueError(f"branching widths must be >= 1, got {list(branching)}")
    return [int(w) for w in branching]


def build_stochastic(prefix, draft, branching, rng: CounterRng, warp: SamplingConfig | None = None,
                     warp_scores: bool = True) -> DraftTree:
    """Sample a draft tree: branching[d] i.i.d. children per node at depth d
    from the (warped) draft distribution; repeats merge (multiplicity)."""
    branching = _check_schedule(branching)
    dm = as_device_model(draft)
    prefix = tuple(int(t) for t in prefix)
    V = dm.vocab_size
    max_nodes = schedule_size(branching)
    session = dm.stochastic_session(prefix, max_nodes, len(branching))
    tree = DraftTree(prefix)
    expandable = 1 + max_nodes - np.prod(branching, dtype=np.int64)  # nodes that can have children
    dev = torch.device("cuda", torch.cuda.current_device())
    qbuf = torch.empty((int(expandable), V), dtype=torch.float64, device=dev)
    dists = DeviceDists(qbuf)
    tree.draft_dists = dists
    temp, top_p = (warp.temperature, warp.top_p) if (warp is not None and warp_scores) else (None, None)
    level = [ROOT]
    for width in branching:
        if not level:
            break
        rows = session.level_rows(tree, level)
        tree.rounds += 1
        n = len(level)
        q0 = len(dists)
        q = qbuf[q0 : q0 + n]
        _scored_rows(rows, q, temp, top_p)
        for j, node in enumerate(level):
            dists.row_of[node] = q0 + j
        u = torch.from_numpy(rng.uniforms(n * width)).to(dev, non_blocking=True)
        ids = torch.arange(q0, q0 + n, dtype=torch.int32, device=dev).repeat_interleave(width)
        tok = torch.empty(n * width, dtype=torch.int32, device=dev)
        logq = torch.empty(n * width, dtype=torch.float64, device=dev)
        _lib.call("sx_sample_rows_idx", _lib.ptr(qbuf), V, V, _lib.ptr(ids), _lib.ptr(u), n * width, _lib.ptr(tok),
                  _lib.ptr(logq), _lib.stream_ptr())
        toks, lq = tok.cpu().tolist(), logq.cpu().tolist()
        K.IO["h2d"] += 8 * n * width
        K.IO["d2h"] += 12 * n * width
        next_level = []
        for j, node in enumerate(level):
            for s in range(j * width, (j + 1) * width):  # tree.py:415-423
                existing = tree.child_with_token(node, toks[s])
                if existing is not None:
                    tree.nodes[existing].multiplicity += 1
                else:
                    next_level.append(tree.add_child(node, toks[s], lq[s]))
        level = next_level
    session.finish(tree)
    return tree


def _scored_rows(rows: torch.Tensor, out: torch.Tensor, temp, top_p) -> None:
    """_scored_dist (tree.py:222-227) of device rows into fp64 out."""
    V = out.shape[1]
    n = out.shape[0]
    if temp is None:  # raw distribution
        if rows.dtype == torch.float64:
            out.copy_(rows[:n])
        else:
            _lib.call("sx_softmax_rows", _lib.ptr(rows), rows.stride(0), V, None, n, _lib.ptr(out), V, _lib.stream_ptr())
        return
    chunk = 64  # bounded warp scratch
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        scratch = K.scratch(_lib.load().sx_warp_scratch_bytes(m, V), out.device, "si_warp")
        _lib.call("sx_warp_rows", _lib.ptr(rows[i : i + m]), K.row_kind(rows), rows.stride(0), V, None, m, float(temp),
                  float(top_p), _lib.ptr(out[i : i + m]), V, _lib.ptr(scratch), _lib.stream_ptr())


def _device_tree(tree: DraftTree, dev):
    n = len(tree.nodes)
    cstart = np.zeros(n + 1, dtype=np.int32)
    ccount = np.zeros(n + 1, dtype=np.int32)
    qrow = np.full(n + 1, -1, dtype=np.int32)
    for r, node in enumerate([ROOT] + list(range(n))):
        ch = tree.children_of(node)
        if ch:
            if ch != list(range(ch[0], ch[0] + len(ch))):
                raise ValueError("stochastic tree children must have consecutive ids")
            cstart[r], ccount[r] = ch[0], len(ch)
        if node in tree.draft_dists:
            qrow[r] = tree.draft_dists.row_of[node]
    tok = np.array([nd.token for nd in tree.nodes] or [0], dtype=np.int32)
    mult = np.array([nd.multiplicity for nd in tree.nodes] or [0], dtype=np.int32)
    return [torch.from_numpy(a).to(dev, non_blocking=True) for a in (qrow, cstart, ccount, tok, mult)]


def verify_specinfer(tree: DraftTree, target, warp: SamplingConfig, rng: CounterRng) -> VerifyOutcome:
    """Multi-round rejection walk over a stochastically drafted tree (specinfer.py:53-96)."""
    if getattr(tree, "draft_dists", None) is None or not isinstance(tree.draft_dists, DeviceDists):
        raise ValueError("tree carries no draft distributions; build it with build_stochastic")
    tm = as_device_model(target)
    rows = tm.tree_rows(tree)
    dev = rows.device
    qrow, cstart, ccount, tok, mult = _device_tree(tree, dev)
    depth = tree.max_depth()
    n_u = sum(nd.multiplicity for nd in tree.nodes) + depth + 2  # upper bound on trials + bonus
    u = torch.from_numpy(rng.peek(n_u)).to(dev, non_blocking=True)
    out = torch.empty(4 + max(depth, 1), dtype=torch.int32, device=dev)
    V = rows.shape[1]
    scratch = K.scratch(_lib.load().sx_row_scratch_bytes(V), dev, "si_verify")
    q = tree.draft_dists.rows
    _lib.call("sx_specinfer_verify", _lib.ptr(rows), K.row_kind(rows), rows.stride(0), V, _lib.ptr(q), q.stride(0),
              _lib.ptr(qrow), _lib.ptr(cstart), _lib.ptr(ccount), _lib.ptr(tok), _lib.ptr(mult), max(depth, 1),
              _lib.ptr(u), n_u, float(warp.temperature), float(warp.top_p), _lib.ptr(out), _lib.ptr(scratch),
              _lib.stream_ptr())
    res = out.cpu().tolist()
    K.IO["h2d"] += 8 * n_u
    K.IO["d2h"] += 4 * len(res)
    plen, bonus, used, err = res[:4]
    if err == 1:
        raise ValueError("rejection residual is not a valid distribution (sampling.py:44-56)")
    if err:
        raise RuntimeError(f"specinfer_verify failed (code {err})")
    rng.counter += used
    tree.target_rows = rows
    return VerifyOutcome(accepted_path=res[4 : 4 + plen], bonus_token=bonus)


def generate_specinfer(prompt, draft, target, branching, cfg: SamplingConfig):
    """Draft-then-verify until cfg.max_new_tokens (specinfer.py:99-127); KV of
    the accepted path is compacted in place for device models with caches."""
    prompt = tuple(int(t) for t in prompt)
    if draft is target and hasattr(target, "draft_view"):
        draft = target.draft_view()  # one network in both roles: a second KV cache for the draft
    rng_draft = CounterRng(cfg.seed, DRAFT_STREAM)
    rng_accept = CounterRng(cfg.seed, ACCEPT_STREAM)
    stats = GenStats()
    tokens: list[int] = []
    while len(tokens) < cfg.max_new_tokens:
        tree = build_stochastic(prompt + tuple(tokens), draft, branching, rng_draft, cfg)
        stats.draft_calls += tree.rounds
        outcome = verify_specinfer(tree, target, cfg, rng_accept)
        stats.target_calls += 1
        emitted = [tree.nodes[i].token for i in outcome.accepted_path]
        emitted.append(outcome.bonus_token)
        emitted = emitted[: cfg.max_new_tokens - len(tokens)]
        _commit(tree, outcome, draft, target)
        tokens.extend(emitted)
        stats.accepted_per_iteration.append(len(emitted))
    stats.tokens_generated = len(tokens)
    return tokens, stats


def _commit(tree, outcome, draft, target) -> None:
    res = SimpleNamespace(path_rows=[i + 1 for i in outcome.accepted_path])
    if hasattr(target, "commit_walk"):
        target.commit_walk(SimpleNamespace(tree=tree, target=target), res)
    if hasattr(draft, "commit_walk") and getattr(tree, "draft_model", None) is draft:
        draft.commit_walk(SimpleNamespace(tree=tree, target=None), res)


def branching_for_budget(budget: int, depth: int) -> list[int]:
    """Stem-shaped schedule with about `budget` nodes (specinfer.py:130-143)."""
    if budget < 1:
        raise ValueError(f"budget must be >= 1, got {budget}")
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    depth = min(depth, budget)
    width = max(1, round(budget / depth))
    return [width] + [1] * (depth - 1)


def schedule_size(branching: list[int]) -> int:
    """Maximum node count a branching schedule can produce (specinfer.py:146-153)."""
    total, level = 0, 1
    for width in branching:
        level *= width
        total += level
    return total
