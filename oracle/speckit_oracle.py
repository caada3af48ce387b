"""CPU oracle: restatement of the reference SpecExec hot path. TEST INFRASTRUCTURE.

Mirrors, function by function, the reference package `speckit` 0.1.0:
  sampling.py  SamplingConfig :21-41, apply_warp :66-98, sample :101-113
  rng.py       CounterRng :32-91 (numpy Philox keyed by sha256(seed \\x1f stream))
  models.py    LanguageModel :32-63, TabularModel :77-97, MarkovModel :100-151,
               make_synthetic :265-279
  tree.py      BuilderParams :36-55, DraftTree :85-205, flatten :208-219,
               build_sssp :240-327
  engine.py    GenStats :30-44, ProbCache :47-70, precompute :73-89,
               generate_specexec :92-131, generate_sequential :134-148,
               stats_record :151-171
The one deliberate deviation is the float64 arithmetic of the scoring / warp /
sample steps, which goes through oracle/oxmath.c (fdlibm log/exp, canonical sum
orders) instead of numpy's dispatch-dependent SIMD routines; see that file's
header. Everything else (ordering keys, heap/threshold bookkeeping, tie-breaks,
RNG streams) follows the reference statements directly.
"""

from __future__ import annotations

import ctypes
import hashlib
import heapq
import json
import math
import pathlib
import subprocess
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIBPATH = _HERE / "liboxref.so"
_lib = None


def build() -> pathlib.Path:
    """Compile oxmath.c (gcc) into oracle/liboxref.so."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIBPATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not _LIBPATH.exists():
            build()
        L = ctypes.CDLL(str(_LIBPATH))
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        L.ox_log.restype = ctypes.c_double
        L.ox_log.argtypes = [ctypes.c_double]
        L.ox_exp.restype = ctypes.c_double
        L.ox_exp.argtypes = [ctypes.c_double]
        L.ox_log_array.argtypes = [dp, dp, ctypes.c_int64]
        L.ox_exp_array.argtypes = [dp, dp, ctypes.c_int64]
        L.ox_canon_sum.restype = ctypes.c_double
        L.ox_canon_sum.argtypes = [dp, ctypes.c_int64]
        L.ox_canon_cumsum.argtypes = [dp, dp, ctypes.c_int64]
        L.ox_softmax_row.argtypes = [fp, ctypes.c_int64, dp]
        L.ox_warp.argtypes = [dp, fp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, dp]
        L.ox_sample.restype = ctypes.c_int64
        L.ox_sample.argtypes = [dp, ctypes.c_int64, ctypes.c_double]
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def ox_log(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().ox_log_array(_dptr(x), _dptr(out), x.size)
    return out


def ox_exp(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().ox_exp_array(_dptr(x), _dptr(out), x.size)
    return out


def canon_sum(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().ox_canon_sum(_dptr(x), x.size))


def canon_cumsum(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().ox_canon_cumsum(_dptr(x), _dptr(out), x.size)
    return out


class Row(np.ndarray):
    """A float64 probability row that remembers the fp32 logits it came from.

    Rows produced by logits-based models (Llama-shaped, replayed GPU rows) carry
    `.logits`; the warp then works from the logits, exactly like the kernels.
    """

    logits: np.ndarray | None = None

    def __array_finalize__(self, obj):
        self.logits = getattr(obj, "logits", None)


def softmax_row(z: np.ndarray) -> Row:
    """Canonical float64 probabilities from fp32 logits: exp(z - max) / S."""
    z = np.ascontiguousarray(z, dtype=np.float32)
    p = np.empty(z.size, dtype=np.float64)
    lib().ox_softmax_row(_fptr(z), z.size, _dptr(p))
    r = p.view(Row)
    r.logits = z
    return r


# ---------------------------------------------------------------------------
# sampling.py
# ---------------------------------------------------------------------------

DIST_ATOL = 1e-9  # sampling.py:18


@dataclass(frozen=True)
class SamplingConfig:
    """sampling.py:21-41"""

    temperature: float = 1.0
    top_p: float = 1.0
    seed: int = 0
    max_new_tokens: int = 16

    def __post_init__(self) -> None:
        if self.temperature < 0:
            raise ValueError(f"temperature must be >= 0, got {self.temperature}")
        if not 0 < self.top_p <= 1:
            raise ValueError(f"top_p must be in (0, 1], got {self.top_p}")
        if self.max_new_tokens < 0:
            raise ValueError(f"max_new_tokens must be >= 0, got {self.max_new_tokens}")


def apply_warp(dist: np.ndarray, cfg: SamplingConfig) -> np.ndarray:
    """sampling.py:66-98 -- t=0 one-hot argmax (lowest id), p**(1/T) renormalised,
    nucleus cut over (p desc, id asc) with the first cumsum >= top_p - 1e-9."""
    z = getattr(dist, "logits", None)
    p = np.ascontiguousarray(dist, dtype=np.float64)
    if cfg.temperature == 1.0 and cfg.top_p >= 1.0:
        return p  # sampling.py:83-98 are no-ops
    out = np.empty(p.size, dtype=np.float64)
    if z is not None:
        z = np.ascontiguousarray(z, dtype=np.float32)
        lib().ox_warp(None, _fptr(z), p.size, float(cfg.temperature), float(cfg.top_p), _dptr(out))
    else:
        lib().ox_warp(_dptr(p), None, p.size, float(cfg.temperature), float(cfg.top_p), _dptr(out))
    return out


def sample(dist: np.ndarray, rng: "CounterRng") -> int:
    """sampling.py:101-113 -- one uniform always consumed; inverse CDF over ids."""
    p = np.ascontiguousarray(dist, dtype=np.float64)
    u = rng.uniform()
    return int(lib().ox_sample(_dptr(p), p.size, u))


# ---------------------------------------------------------------------------
# rng.py
# ---------------------------------------------------------------------------

_BLOCK = 1024  # rng.py:23


def _stream_key(seed: int, stream: str) -> int:
    """rng.py:26-29"""
    digest = hashlib.sha256(f"{seed}\x1f{stream}".encode()).digest()
    return int.from_bytes(digest[:16], "little")


class CounterRng:
    """rng.py:32-91 -- n-th draw of Philox(key) `Generator.random()`."""

    def __init__(self, seed: int, stream: str = "generation", counter: int = 0) -> None:
        if counter < 0:
            raise ValueError(f"counter must be >= 0, got {counter}")
        self.seed = int(seed)
        self.stream = stream
        self.counter = int(counter)
        self._key = _stream_key(self.seed, stream)
        self._gen = None
        self._buffer = np.empty(0, dtype=np.float64)

    def _ensure(self, n: int) -> None:
        if n < self._buffer.size:
            return
        if self._gen is None:
            self._gen = np.random.Generator(np.random.Philox(key=self._key))
        size = max(64, min(2 * self._buffer.size, _BLOCK * 64))
        while size <= n:
            size *= 2
        self._buffer = np.concatenate([self._buffer, self._gen.random(size - self._buffer.size)])

    def draw_at(self, index: int) -> float:
        if index < 0:
            raise ValueError(f"index must be >= 0, got {index}")
        self._ensure(index)
        return float(self._buffer[index])

    def uniform(self) -> float:
        value = self.draw_at(self.counter)
        self.counter += 1
        return value

    def uniforms(self, n: int) -> np.ndarray:
        if n < 0:
            raise ValueError(f"n must be >= 0, got {n}")
        self._ensure(self.counter + n)
        out = self._buffer[self.counter : self.counter + n].copy()
        self.counter += n
        return out


# ---------------------------------------------------------------------------
# models.py
# ---------------------------------------------------------------------------

Prefix = tuple[int, ...]


def _check_prefix(prefix: Sequence[int], vocab_size: int) -> Prefix:
    """models.py:24-29"""
    toks = tuple(int(t) for t in prefix)
    for t in toks:
        if not 0 <= t < vocab_size:
            raise ValueError(f"token id {t} outside vocabulary [0, {vocab_size})")
    return toks


class LanguageModel:
    """models.py:32-63"""

    vocab_size: int
    backend: str

    def next_distribution(self, prefix: Sequence[int]) -> np.ndarray:
        raise NotImplementedError

    def next_distributions(self, prefixes: Iterable[Sequence[int]]) -> np.ndarray:
        rows = [self.next_distribution(p) for p in prefixes]
        if not rows:
            return np.empty((0, self.vocab_size))
        return rows  # list of rows (each may carry .logits)


def _normalize_rows(table: np.ndarray) -> np.ndarray:
    """models.py:66-74"""
    table = np.asarray(table, dtype=np.float64)
    sums = table.sum(axis=-1, keepdims=True)
    if np.any(table < 0) or np.any(sums <= 0):
        raise ValueError("probability table rows must be non-negative with positive mass")
    if np.max(np.abs(sums - 1.0)) <= 1e-9:
        return table.copy()
    return table / sums


class TabularModel(LanguageModel):
    """models.py:77-97"""

    backend = "tabular"

    def __init__(self, row: Sequence[float]) -> None:
        self.row = _normalize_rows(np.asarray(row, dtype=np.float64)[None, :])[0]
        self.vocab_size = self.row.size

    def next_distribution(self, prefix):
        _check_prefix(prefix, self.vocab_size)
        return self.row.copy()

    def power_smoothed(self, power: float) -> "TabularModel":
        return TabularModel(self.row**power)


class MarkovModel(LanguageModel):
    """models.py:100-151 -- context = last `order` tokens, left-padded with 0."""

    backend = "markov"

    def __init__(self, table: np.ndarray, order: int = 1) -> None:
        if order < 1:
            raise ValueError(f"order must be >= 1, got {order}")
        table = _normalize_rows(table)
        vocab = table.shape[1]
        if table.shape[0] != vocab**order:
            raise ValueError(f"table has {table.shape[0]} rows, expected vocab**order = {vocab**order}")
        self.table = table
        self.order = order
        self.vocab_size = vocab

    def _row_index(self, prefix: Prefix) -> int:
        context = prefix[-self.order :]
        context = (0,) * (self.order - len(context)) + context
        idx = 0
        for t in context:
            idx = idx * self.vocab_size + t
        return idx

    def next_distribution(self, prefix):
        toks = _check_prefix(prefix, self.vocab_size)
        return self.table[self._row_index(toks)].copy()

    def power_smoothed(self, power: float) -> "MarkovModel":
        return MarkovModel(self.table**power, order=self.order)


def make_synthetic(seed: int, vocab_size: int, sharpness: float, order: int = 1) -> MarkovModel:
    """models.py:265-279"""
    if vocab_size < 2:
        raise ValueError(f"vocab_size must be >= 2, got {vocab_size}")
    if sharpness <= 0:
        raise ValueError(f"sharpness must be > 0, got {sharpness}")
    gen = np.random.default_rng(seed)
    table = gen.dirichlet(np.full(vocab_size, sharpness), size=vocab_size**order)
    return MarkovModel(table, order=order)


class LogitsLM(LanguageModel):
    """A logits-producing model (Llama-shaped or synthetic): rows are canonical
    float64 softmax of fp32 logits, carrying the logits for the warp."""

    backend = "logits"

    def __init__(self, vocab_size: int, logits_fn: Callable[[list[Prefix]], np.ndarray]) -> None:
        self.vocab_size = vocab_size
        self.logits_fn = logits_fn

    def next_distribution(self, prefix):
        return self.next_distributions([prefix])[0]

    def next_distributions(self, prefixes):
        prefixes = [tuple(int(t) for t in p) for p in prefixes]
        if not prefixes:
            return np.empty((0, self.vocab_size))
        z = np.asarray(self.logits_fn(prefixes), dtype=np.float32)
        return [softmax_row(z[i]) for i in range(len(prefixes))]


def hashed_logits_fn(vocab: int, seed: int, scale: float = 1.3, bias_table: np.ndarray | None = None):
    """Deterministic synthetic logits keyed by the prefix (stands in for a model
    whose rows are replayed). fp32 logits ~ N(0, scale) from a per-prefix seed;
    `bias_table[last_token]` (optional) adds a shared bigram bias."""

    def fn(prefixes):
        out = np.empty((len(prefixes), vocab), dtype=np.float32)
        for i, p in enumerate(prefixes):
            h = hashlib.sha256((f"{seed}:" + ",".join(map(str, p))).encode()).digest()
            g = np.random.default_rng(int.from_bytes(h[:8], "little"))
            z = g.standard_normal(vocab, dtype=np.float32) * np.float32(scale)
            if bias_table is not None and p:
                z = z + bias_table[p[-1] % bias_table.shape[0]]
            out[i] = z
        return out

    return fn


# ---------------------------------------------------------------------------
# tree.py
# ---------------------------------------------------------------------------

ROOT = -1  # tree.py:33


@dataclass(frozen=True)
class BuilderParams:
    """tree.py:36-55"""

    budget: int
    max_depth: int
    batch_size: int = 8

    def __post_init__(self) -> None:
        if self.budget < 1:
            raise ValueError(f"budget must be >= 1, got {self.budget}")
        if self.max_depth < 1:
            raise ValueError(f"max_depth must be >= 1, got {self.max_depth}")
        if self.batch_size < 1:
            raise ValueError(f"batch_size must be >= 1, got {self.batch_size}")


@dataclass
class DraftNode:
    """tree.py:58-68"""

    node_id: int
    parent: int
    token: int
    edge_logprob: float
    cum_logprob: float
    depth: int
    multiplicity: int = 1


@dataclass
class FlattenedTree:
    """tree.py:71-82"""

    order: list[int]
    ancestor_mask: np.ndarray


class DraftTree:
    """tree.py:85-205 (the subset the hot path and the parity tests use)."""

    def __init__(self, prefix: Prefix) -> None:
        self.prefix: Prefix = tuple(prefix)
        self.nodes: list[DraftNode] = []
        self.rounds = 0
        self._children: dict[int, list[int]] = {ROOT: []}

    def __len__(self) -> int:
        return len(self.nodes)

    def add_child(self, parent: int, token: int, edge_logprob: float) -> int:
        """tree.py:104-121"""
        if parent != ROOT and not 0 <= parent < len(self.nodes):
            raise KeyError(f"no node with id {parent}")
        node_id = len(self.nodes)
        parent_cum = 0.0 if parent == ROOT else self.nodes[parent].cum_logprob
        parent_depth = 0 if parent == ROOT else self.nodes[parent].depth
        self.nodes.append(
            DraftNode(node_id, parent, int(token), float(edge_logprob), parent_cum + float(edge_logprob), parent_depth + 1)
        )
        self._children[node_id] = []
        self._children[parent].append(node_id)
        return node_id

    def children_of(self, node_id: int) -> list[int]:
        return list(self._children[node_id])

    def child_with_token(self, node_id: int, token: int) -> int | None:
        """tree.py:132-136"""
        for child in self._children[node_id]:
            if self.nodes[child].token == token:
                return child
        return None

    def path_tokens(self, node_id: int) -> Prefix:
        """tree.py:138-148"""
        if node_id == ROOT:
            return ()
        path = []
        while node_id != ROOT:
            node = self.nodes[node_id]
            path.append(node.token)
            node_id = node.parent
        return tuple(reversed(path))

    def full_prefix(self, node_id: int) -> Prefix:
        return self.prefix + self.path_tokens(node_id)

    def max_depth(self) -> int:
        return max((n.depth for n in self.nodes), default=0)

    def to_json(self) -> str:
        """tree.py:175-191"""
        return json.dumps(
            {
                "prefix": list(self.prefix),
                "nodes": [
                    {
                        "id": n.node_id,
                        "parent": n.parent,
                        "token": n.token,
                        "edge_logprob": n.edge_logprob,
                        "cum_logprob": n.cum_logprob,
                    }
                    for n in self.nodes
                ],
            }
        )


def flatten(tree: DraftTree) -> FlattenedTree:
    """tree.py:208-219"""
    order = [n.node_id for n in tree.nodes]
    m = len(order) + 1
    mask = np.zeros((m, m), dtype=bool)
    mask[0, 0] = True
    for node in tree.nodes:
        pos = node.node_id + 1
        mask[pos] = mask[node.parent + 1]
        mask[pos, pos] = True
    return FlattenedTree(order=order, ancestor_mask=mask)


def _scored_dist(dist, warp, warp_scores):
    """tree.py:222-227"""
    if warp is not None and warp_scores:
        return apply_warp(dist, warp)
    return np.asarray(dist, dtype=np.float64)


def build_sssp(
    prefix: Prefix,
    draft: LanguageModel,
    params: BuilderParams,
    warp: SamplingConfig | None = None,
    warp_scores: bool = True,
) -> DraftTree:
    """tree.py:240-327, statement by statement.

    One exact shortcut: before the per-round sort (tree.py:309) each row keeps
    only its `budget` best children by (nll, token) -- within a row depth and
    parent path are shared, so no child outside that set can reach
    children[:budget].
    """
    tree = DraftTree(prefix)
    budget, max_depth, batch = params.budget, params.max_depth, params.batch_size
    materialized: dict[Prefix, tuple[float, int, float]] = {}
    heap: list[tuple[float, int, Prefix, float]] = []
    threshold = None

    def prune_materialized() -> None:  # tree.py:270-278
        nonlocal materialized, threshold
        if len(materialized) >= budget:
            items = sorted(materialized.items(), key=lambda kv: (kv[1][0], kv[1][1], kv[0]))[:budget]
            materialized = dict(items)
            worst_path, (worst_nll, worst_depth, _) = items[-1]
            threshold = (worst_nll, worst_depth, worst_path)

    pending_root = True
    while True:  # tree.py:281-318
        batch_paths: list[Prefix] = []
        if pending_root:
            batch_paths.append(())
            pending_root = False
        while len(batch_paths) < batch and heap:
            nll, depth, path, _ = heap[0]
            if threshold is not None and (nll, depth, path) >= threshold:
                break
            heapq.heappop(heap)
            if depth < max_depth:
                batch_paths.append(path)
        if not batch_paths:
            break

        dists = draft.next_distributions([prefix + p for p in batch_paths])
        tree.rounds += 1

        children: list[tuple[float, int, Prefix, float]] = []
        for path, dist in zip(batch_paths, dists):
            scored = _scored_dist(dist, warp, warp_scores)
            parent_nll = 0.0 if not path else materialized[path][0]
            toks = np.nonzero(scored > 0)[0]
            edges = ox_log(scored[toks])
            nlls = parent_nll - edges
            if toks.size > budget:
                keep = np.lexsort((toks, nlls))[:budget]
                toks, edges, nlls = toks[keep], edges[keep], nlls[keep]
            depth = len(path) + 1
            for t, e, n in zip(toks.tolist(), edges.tolist(), nlls.tolist()):
                children.append((n, depth, path + (t,), e))

        children.sort(key=lambda c: (c[0], c[1], c[2]))
        for nll, depth, path, edge in children[:budget]:
            materialized[path] = (nll, depth, edge)
            heapq.heappush(heap, (nll, depth, path, edge))
        prune_materialized()
        if len(heap) > budget:
            heap = heapq.nsmallest(budget, heap)
            heapq.heapify(heap)

    final = sorted(materialized.items(), key=lambda kv: (kv[1][0], kv[1][1], kv[0]))
    path_to_id: dict[Prefix, int] = {(): ROOT}
    for path, (_, _, edge) in final[:budget]:
        parent_id = path_to_id[path[:-1]]
        path_to_id[path] = tree.add_child(parent_id, path[-1], edge)
    return tree


# ---------------------------------------------------------------------------
# engine.py
# ---------------------------------------------------------------------------

GENERATION_STREAM = "generation"  # engine.py:27


@dataclass
class GenStats:
    """engine.py:30-44"""

    target_calls: int = 0
    draft_calls: int = 0
    tokens_generated: int = 0
    accepted_per_iteration: list[int] = field(default_factory=list)

    @property
    def generation_rate(self) -> float:
        if self.target_calls == 0:
            return 0.0
        return self.tokens_generated / self.target_calls


class ProbCache:
    """engine.py:47-70"""

    def __init__(self, prefix, tree, dists) -> None:
        self.prefix = prefix
        self.tree = tree
        self.dists = dists
        self.cursor = ROOT

    def current_dist(self):
        return self.dists[self.cursor + 1]

    def advance(self, token: int) -> bool:
        child = self.tree.child_with_token(self.cursor, token)
        if child is None:
            return False
        self.cursor = child
        return True


def precompute(prefix, draft, target, params, warp=None, warp_scores: bool = True) -> ProbCache:
    """engine.py:73-89 (warp_scores: SURVEY F2 builder flag, default = reference)."""
    tree = build_sssp(prefix, draft, params, warp, warp_scores)
    flat = flatten(tree)
    prefixes = [prefix] + [tree.full_prefix(i) for i in flat.order]
    dists = target.next_distributions(prefixes)
    return ProbCache(prefix, tree, dists)


def generate_specexec(prompt, draft, target, params, cfg, warp_scores: bool = True):
    """engine.py:92-131"""
    prompt = tuple(prompt)
    rng = CounterRng(cfg.seed, GENERATION_STREAM)
    stats = GenStats()
    tokens: list[int] = []
    if cfg.max_new_tokens == 0:
        return tokens, stats
    cache = precompute(prompt, draft, target, params, cfg, warp_scores)
    stats.target_calls += 1
    stats.draft_calls += cache.tree.rounds
    stats.accepted_per_iteration.append(0)
    for _ in range(cfg.max_new_tokens):
        if cache is None:
            cache = precompute(prompt + tuple(tokens), draft, target, params, cfg, warp_scores)
            stats.target_calls += 1
            stats.draft_calls += cache.tree.rounds
            stats.accepted_per_iteration.append(0)
        token = sample(apply_warp(cache.current_dist(), cfg), rng)
        tokens.append(token)
        stats.accepted_per_iteration[-1] += 1
        if not cache.advance(token):
            cache = None
    stats.tokens_generated = len(tokens)
    return tokens, stats


def generate_sequential(prompt, target, cfg):
    """engine.py:134-148"""
    prompt = tuple(prompt)
    rng = CounterRng(cfg.seed, GENERATION_STREAM)
    stats = GenStats()
    tokens: list[int] = []
    for _ in range(cfg.max_new_tokens):
        dist = target.next_distribution(prompt + tuple(tokens))
        tokens.append(sample(apply_warp(dist, cfg), rng))
        stats.target_calls += 1
        stats.accepted_per_iteration.append(1)
    stats.tokens_generated = len(tokens)
    return tokens, stats


def stats_record(method, cfg, stats, budget, depth, batch_size) -> dict:
    """engine.py:151-171"""
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


def tree_topology(tree) -> list[tuple[int, int]]:
    """(parent, token) per node id: the integer part parity is asserted on."""
    return [(n.parent, n.token) for n in tree.nodes]


# ---------------------------------------------------------------------------
# specinfer.py + tree.py build_stochastic (the SpecInfer baseline)
# ---------------------------------------------------------------------------

SI_DRAFT_STREAM = "specinfer-draft"  # specinfer.py:26
SI_ACCEPT_STREAM = "specinfer-accept"  # specinfer.py:27


def _log_edges(q: np.ndarray) -> np.ndarray:
    """tree.py:230-232 -- log of the scored distribution, zero -> -inf."""
    out = np.full(q.shape, -np.inf)
    nz = q > 0
    out[nz] = ox_log(q[nz])
    return out


def build_stochastic(prefix, draft, branching, rng, warp=None, warp_scores: bool = True) -> DraftTree:
    """tree.py:383-425 -- branching[d] i.i.d. samples per node at depth d from the
    (warped) draft distribution; repeats merge into one node with multiplicity;
    the sampled-from distribution of every expanded node is kept."""
    if not branching:
        raise ValueError("branching schedule must be non-empty")
    if any(w < 1 for w in branching):
        raise ValueError(f"branching widths must be >= 1, got {branching}")
    tree = DraftTree(prefix)
    tree.draft_dists = {}
    level = [ROOT]
    for width in branching:
        if not level:
            break
        dists = draft.next_distributions([tree.full_prefix(n) for n in level])
        tree.rounds += 1
        next_level = []
        for node_id, dist in zip(level, dists):
            q = _scored_dist(dist, warp, warp_scores)
            tree.draft_dists[node_id] = q
            log_q = _log_edges(q)
            for _ in range(width):
                token = sample(q, rng)
                existing = tree.child_with_token(node_id, token)
                if existing is not None:
                    tree.nodes[existing].multiplicity += 1
                else:
                    next_level.append(tree.add_child(node_id, token, float(log_q[token])))
        level = next_level
    return tree


def validate_distribution(p: np.ndarray) -> np.ndarray:
    """sampling.py:44-56 (sum in the canonical order)."""
    p = np.asarray(p, dtype=np.float64)
    if p.ndim != 1 or p.size == 0:
        raise ValueError("distribution must be a non-empty 1-D array")
    if np.any(p < 0):
        raise ValueError("distribution has negative entries")
    total = canon_sum(p)
    if abs(total - 1.0) > DIST_ATOL:
        raise ValueError(f"distribution sums to {total!r}, expected 1 within {DIST_ATOL}")
    return p


def residual(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """specinfer.py:42-50 -- normalize(max(p - q, 0)); p itself when nothing is left."""
    diff = np.maximum(p - q, 0.0)
    total = canon_sum(diff)
    if total <= 0.0:
        return np.array(p, dtype=np.float64, copy=True)
    return validate_distribution(diff / total)


@dataclass
class VerifyOutcome:
    """specinfer.py:30-39"""

    accepted_path: list[int]
    bonus_token: int

    @property
    def tokens_emitted(self) -> int:
        return len(self.accepted_path) + 1


def verify_specinfer(tree: DraftTree, target, warp: SamplingConfig, rng: CounterRng) -> VerifyOutcome:
    """specinfer.py:53-96 -- multi-round rejection walk: child after child (each
    `multiplicity` times) is accepted with probability min(1, p[x]/q[x]); a
    rejection moves p to the residual; no acceptance -> bonus token from p."""
    if getattr(tree, "draft_dists", None) is None:
        raise ValueError("tree carries no draft distributions; build it with build_stochastic")
    flat = flatten(tree)
    prefixes = [tree.prefix] + [tree.full_prefix(i) for i in flat.order]
    target_dists = target.next_distributions(prefixes)
    node = ROOT
    path: list[int] = []
    p = apply_warp(target_dists[0], warp)
    while True:
        accepted = None
        for child_id in tree.children_of(node):
            child = tree.nodes[child_id]
            q = tree.draft_dists[node]
            for _ in range(child.multiplicity):
                ratio = min(1.0, p[child.token] / q[child.token])
                if rng.uniform() < ratio:
                    accepted = child_id
                    break
                p = residual(p, q)
            if accepted is not None:
                break
        if accepted is None:
            return VerifyOutcome(accepted_path=path, bonus_token=sample(p, rng))
        path.append(accepted)
        node = accepted
        p = apply_warp(target_dists[accepted + 1], warp)


def generate_specinfer(prompt, draft, target, branching, cfg: SamplingConfig):
    """specinfer.py:99-127"""
    prompt = tuple(prompt)
    rng_draft = CounterRng(cfg.seed, SI_DRAFT_STREAM)
    rng_accept = CounterRng(cfg.seed, SI_ACCEPT_STREAM)
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
        tokens.extend(emitted)
        stats.accepted_per_iteration.append(len(emitted))
    stats.tokens_generated = len(tokens)
    return tokens, stats


def branching_for_budget(budget: int, depth: int) -> list[int]:
    """specinfer.py:130-143 -- `width` stems of length `depth`."""
    if budget < 1:
        raise ValueError(f"budget must be >= 1, got {budget}")
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    depth = min(depth, budget)
    width = max(1, round(budget / depth))
    return [width] + [1] * (depth - 1)


def schedule_size(branching: list[int]) -> int:
    """specinfer.py:146-153"""
    total, level = 0, 1
    for width in branching:
        level *= width
        total += level
    return total


# ---------------------------------------------------------------------------
# tree.py build_beam (Appendix F ablation)
# ---------------------------------------------------------------------------


def build_beam(prefix, draft, beam_size: int, max_len: int, warp=None, warp_scores: bool = True) -> DraftTree:
    """tree.py:330-380 -- standard beam search under (nll, path); the tree is the
    prefix closure of the final beam, node ids in (length, path) order.

    One exact shortcut: each beam row contributes only its `beam_size` best
    candidates by (nll, token) -- within a row the path prefix is shared, so no
    other candidate of that row can reach the global top `beam_size`."""
    if beam_size < 1:
        raise ValueError(f"beam_size must be >= 1, got {beam_size}")
    if max_len < 1:
        raise ValueError(f"max_len must be >= 1, got {max_len}")
    tree = DraftTree(prefix)
    beams: list[tuple[float, Prefix]] = [(0.0, ())]
    edges: dict[Prefix, float] = {}
    for _ in range(max_len):
        dists = draft.next_distributions([tuple(prefix) + path for _, path in beams])
        tree.rounds += 1
        candidates = []
        for (nll, path), dist in zip(beams, dists):
            scored = _scored_dist(dist, warp, warp_scores)
            toks = np.nonzero(scored > 0)[0]
            edge = ox_log(scored[toks])
            cn = nll - edge
            if toks.size > beam_size:
                keep = np.lexsort((toks, cn))[:beam_size]
                toks, edge, cn = toks[keep], edge[keep], cn[keep]
            for t, e, c in zip(toks.tolist(), edge.tolist(), cn.tolist()):
                candidates.append((c, path + (int(t),), e))
        if not candidates:
            break
        candidates.sort(key=lambda c: (c[0], c[1]))
        kept = candidates[:beam_size]
        for _, path, edge in kept:
            edges[path] = edge
        beams = [(nll, path) for nll, path, _ in kept]
    keep: set[Prefix] = set()
    for _, path in beams:
        for end in range(1, len(path) + 1):
            keep.add(path[:end])
    path_to_id: dict[Prefix, int] = {(): ROOT}
    for path in sorted(keep, key=lambda p: (len(p), p)):
        path_to_id[path] = tree.add_child(path_to_id[path[:-1]], path[-1], edges[path])
    return tree
