"""SpecExec generation on the GPU: precompute + the acceptance walk.

API of the reference engine (pkg/src/speckit/engine.py): `GenStats` (:30-44),
`ProbCache` (:47-70), `precompute` (:73-89), `generate_specexec` (:92-131),
`generate_sequential` (:134-148), `stats_record` (:151-171).

One target iteration = `precompute` (GPU tree build, then ONE target pass over
the anchor + every tree node, rows kept on the device) followed by the walk
kernel, which consumes the cached rows exactly like the reference loop
(sample(apply_warp(row), u), advance to the child carrying the token, stop on a
miss) with the uniforms of the same CounterRng "generation" stream. Because the
cache holds the target's raw rows and the warp is applied at draw time, the
output equals `generate_sequential` for every seed.

`generate_specexec` resolves `precompute` through this module's globals, so a
monkeypatched precompute (fault injection, pkg/tests/test_harness.py:301-316)
is honoured.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .models import as_device_model
from .rng import CounterRng
from .sampling import SamplingConfig
from .tree import ROOT, BuilderParams, DraftTree, build_sssp

GENERATION_STREAM = "generation"


@dataclass
class GenStats:
    """Call accounting for one generation run (engine.py:30-44)."""

    target_calls: int = 0
    draft_calls: int = 0
    tokens_generated: int = 0
    accepted_per_iteration: list[int] = field(default_factory=list)

    @property
    def generation_rate(self) -> float:
        if self.target_calls == 0:
            return 0.0
        return self.tokens_generated / self.target_calls


class RowView(np.ndarray):
    """A float64 row materialised from the device cache; remembers its source."""

    _src = None


class DeviceRows:
    """`ProbCache.dists` kept in HBM (fp32 logits or fp64 probabilities).

    Indexing materialises the float64 row on demand (only the <= D+1 rows the
    walk touches are ever needed; the dense [K+1, V] float64 matrix of the
    reference is never built). Assigning a row copies device rows (used by the
    fault-injection tests)."""

    def __init__(self, rows: torch.Tensor):
        self.rows = rows

    @property
    def shape(self):
        return tuple(self.rows.shape)

    def __len__(self):
        return self.rows.shape[0]

    def row_tensor(self, i: int) -> torch.Tensor:
        return self.rows[i]

    def __getitem__(self, i):
        if isinstance(i, tuple) or not isinstance(i, (int, np.integer)):
            return np.stack([self[j] for j in range(len(self))])[i]
        i = int(i)
        if self.rows.dtype == torch.int64:
            raise RuntimeError("argmax-only target rows (LlamaModel(tp_argmax=True), KV1): the full distribution "
                               "is not kept -- build the target without tp_argmax to read rows")
        if self.rows.dtype == torch.float32:
            r = K.softmax_rows(self.rows[i : i + 1])[0]
        else:
            r = self.rows[i]
        out = r.cpu().numpy().view(RowView)
        out._src = (self, i)
        return out

    def __setitem__(self, i, value):
        src = getattr(value, "_src", None)
        if src is not None and src[0].rows.dtype == self.rows.dtype:
            self.rows[int(i)].copy_(src[0].rows[src[1]])
            return
        v = torch.as_tensor(np.asarray(value, dtype=np.float64), device=self.rows.device)
        if self.rows.dtype == torch.float32:
            v = torch.where(v > 0, v.log(), torch.full_like(v, -1e30)).float()
        self.rows[int(i)].copy_(v)

    def __array__(self, dtype=None, copy=None):
        a = self[slice(None)]
        return a.astype(dtype) if dtype is not None else a


class ProbCache:
    """Target rows for every prefix in a draft tree (engine.py:47-70).

    Row 0 is the anchor's distribution, row i+1 node i's; the cursor starts at
    the root. `walk` runs the device acceptance walk from the cursor."""

    def __init__(self, prefix, tree: DraftTree, dists, target=None) -> None:
        self.prefix = prefix
        self.tree = tree
        self.dists = dists if isinstance(dists, DeviceRows) else DeviceRows(dists)
        self.cursor = ROOT
        self.target = target

    def current_dist(self) -> np.ndarray:
        return self.dists[self.cursor + 1]

    def advance(self, token: int) -> bool:
        child = self.tree.child_with_token(self.cursor, token)
        if child is None:
            return False
        self.cursor = child
        return True

    def _device_tree(self):
        t = self.tree
        if t.device_parent is None:
            dev = self.dists.rows.device
            t.device_parent = torch.tensor([n.parent for n in t.nodes] or [0], dtype=torch.int32, device=dev)
            t.device_token = torch.tensor([n.token for n in t.nodes] or [0], dtype=torch.int32, device=dev)
        return t.device_parent, t.device_token

    def walk(self, uniforms: np.ndarray, cfg: SamplingConfig, max_steps: int) -> K.WalkResult:
        parent, token = self._device_tree()
        res = K.verify_walk(self.dists.rows, parent, token, len(self.tree.nodes), self.cursor, uniforms, max_steps,
                            cfg.temperature, cfg.top_p)
        if not res.fell_off:
            self.cursor = res.cursor
        return res


def precompute(
    prefix,
    draft,
    target,
    params: BuilderParams,
    warp: SamplingConfig | None = None,
    warp_scores: bool = True,
) -> ProbCache:
    """Build the draft tree on the GPU and fill the cache with ONE target pass
    over the anchor and every node (engine.py:73-89). `warp_scores=False`
    scores the tree with the raw draft distribution (SURVEY F2 builder flag)."""
    prefix = tuple(int(t) for t in prefix)
    _mark("draft")
    tree = build_sssp(prefix, draft, params, warp, warp_scores)
    _mark("target")
    rows = as_device_model(target).tree_rows(tree)
    _mark("verify")
    return ProbCache(prefix, tree, rows, target)


class StageTimer:
    """CUDA events at stage boundaries on the current stream (bench.py breakdown)."""

    def __init__(self):
        self.marks: list[tuple[str, torch.cuda.Event]] = []

    def mark(self, name: str) -> None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e))

    def totals(self) -> dict[str, float]:
        torch.cuda.synchronize()
        out: dict[str, float] = {}
        for (name, e0), (_, e1) in zip(self.marks, self.marks[1:]):
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        return out


STAGES: StageTimer | None = None


def _mark(name: str) -> None:
    if STAGES is not None:
        STAGES.mark(name)


def _max_walk(cache: ProbCache) -> int:
    # from the cursor the walk can emit at most (remaining depth) + 1 tokens
    t = cache.tree
    d0 = 0 if cache.cursor == ROOT else t.nodes[cache.cursor].depth
    return t.max_depth() - d0 + 1


class SpecExecSession:
    """Iteration-level driver of generate_specexec: each `step()` is one target
    iteration (precompute if the previous token fell off the tree, then the
    device walk until a miss or the token limit)."""

    def __init__(self, prompt, draft, target, params: BuilderParams, cfg: SamplingConfig, warp_scores: bool = True):
        if draft is target and hasattr(target, "draft_view"):
            draft = target.draft_view()  # one network in both roles: a second KV cache for the draft
        self.prompt = tuple(int(t) for t in prompt)
        self.draft, self.target, self.params, self.cfg = draft, target, params, cfg
        self.warp_scores = warp_scores
        self.rng = CounterRng(cfg.seed, GENERATION_STREAM)
        self.stats = GenStats()
        self.tokens: list[int] = []
        self.cache: ProbCache | None = None

    def _precompute(self) -> ProbCache:
        prefix = self.prompt + tuple(self.tokens)
        # resolved through the module global (fault-injection tests monkeypatch it)
        if self.warp_scores:
            cache = precompute(prefix, self.draft, self.target, self.params, self.cfg)
        else:
            cache = precompute(prefix, self.draft, self.target, self.params, self.cfg, warp_scores=False)
        self.stats.target_calls += 1
        self.stats.draft_calls += cache.tree.rounds
        self.stats.accepted_per_iteration.append(0)
        return cache

    def step(self, limit: int) -> list[int]:
        """Emit up to `limit` tokens from one target iteration."""
        if self.cache is None:
            self.cache = self._precompute()
        cache = self.cache
        steps = min(limit, _max_walk(cache))
        res = cache.walk(self.rng.peek(steps), self.cfg, steps)
        self.rng.counter += len(res.tokens)
        self.tokens.extend(res.tokens)
        self.stats.accepted_per_iteration[-1] += len(res.tokens)
        self.stats.tokens_generated = len(self.tokens)
        if res.fell_off:
            if hasattr(self.target, "commit_walk"):
                self.target.commit_walk(cache, res)
            if hasattr(self.draft, "commit_walk"):
                self.draft.commit_walk(cache, res)
            self.cache = None
        _mark("host")
        return res.tokens


def generate_specexec(prompt, draft, target, params: BuilderParams, cfg: SamplingConfig, warp_scores: bool = True):
    """Decode with the speculative cache; equal to `generate_sequential` (engine.py:92-131)."""
    sess = SpecExecSession(prompt, draft, target, params, cfg, warp_scores)
    if cfg.max_new_tokens == 0:
        return sess.tokens, sess.stats
    sess.cache = sess._precompute()  # first iteration before the loop (engine.py:113-116)
    while len(sess.tokens) < cfg.max_new_tokens:
        sess.step(cfg.max_new_tokens - len(sess.tokens))
    sess.stats.tokens_generated = len(sess.tokens)
    return sess.tokens, sess.stats


def generate_sequential(prompt, target, cfg: SamplingConfig):
    """One token at a time (engine.py:134-148): one target row per token, the
    same warp + sample kernels and the same uniform stream."""
    prompt = tuple(int(t) for t in prompt)
    rng = CounterRng(cfg.seed, GENERATION_STREAM)
    stats = GenStats()
    tokens: list[int] = []
    tm = as_device_model(target)
    empty_parent = None
    for _ in range(cfg.max_new_tokens):
        rows = tm.prefix_rows(prompt + tuple(tokens))
        if empty_parent is None:
            empty_parent = torch.zeros(1, dtype=torch.int32, device=rows.device)
        res = K.verify_walk(rows, empty_parent, empty_parent, 0, ROOT, rng.peek(1), 1, cfg.temperature, cfg.top_p)
        rng.counter += 1
        tokens.append(res.tokens[0])
        stats.target_calls += 1
        stats.accepted_per_iteration.append(1)
    stats.tokens_generated = len(tokens)
    return tokens, stats


def stats_record(method: str, cfg: SamplingConfig, stats: GenStats, budget: int, depth: int, batch_size: int) -> dict:
    """Per-run stats record in the shared JSON-lines schema (engine.py:151-171)."""
    return {
        "method": method,
        "K": budget,
        "D": depth,
        "B": batch_size,
        "t": cfg.temperature,
        "top_p": cfg.top_p,
        "seed": cfg.seed,
        "tokens": stats.tokens_generated,
        "target_calls": stats.target_calls,
        "generation_rate": stats.generation_rate,
    }
