"""Language-model plugins: the reference interface over device-resident models.

`LanguageModel` is the reference plugin API (pkg/src/speckit/models.py:32-63):
`vocab_size`, `backend`, `next_distribution(prefix) -> float64[V]` and
`next_distributions(prefixes) -> float64[n, V]`, pure and batch-consistent,
`ValueError` on out-of-vocabulary tokens (:24-29).

Every model in this package is additionally a *device model*: it keeps its
parameters in HBM and produces next-token rows for draft-tree nodes directly on
the GPU (no host round trip per row), which is what the GPU tree builder and
the target pass over the tree consume:

  tree_session(prefix, params) -> session with .ws (TreeWorkspace), .batch_rows(),
                                  .advance(ctl), .finish(tree)
  tree_rows(tree) -> device rows [len(tree)+1, V] (row 0 = anchor, row i+1 = node i)

The exact table backends (`TabularModel`, `MarkovModel`, `make_synthetic`,
models.py:77-151, 265-279) upload their float64 tables; Llama-shaped models live
in `llama.py`.
"""

from __future__ import annotations

import json
import threading
import weakref
from typing import Iterable, Sequence

import numpy as np
import torch

from . import kernels as K
from .tree import BuilderParams

Prefix = tuple[int, ...]


def _check_prefix(prefix: Sequence[int], vocab_size: int) -> Prefix:
    toks = tuple(int(t) for t in prefix)
    for t in toks:
        if not 0 <= t < vocab_size:
            raise ValueError(f"token id {t} outside vocabulary [0, {vocab_size})")
    return toks


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2406_02532_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


class LanguageModel:
    """Interface shared by all backends (models.py:32-63)."""

    vocab_size: int
    backend: str

    def next_distribution(self, prefix: Sequence[int]) -> np.ndarray:
        return self.next_distributions([prefix])[0]

    def next_distributions(self, prefixes: Iterable[Sequence[int]]) -> np.ndarray:
        raise NotImplementedError

    def to_json(self) -> str:
        raise NotImplementedError

    def decode(self, tokens: Sequence[int]) -> str:
        return " ".join(str(int(t)) for t in tokens)

    def encode(self, text: str) -> Prefix:
        raise NotImplementedError(f"{self.backend} backend has no text mapping")


def as_device_model(model) -> "LanguageModel":
    """The device-model view of a plugin: this package's models as they are; any
    other object with the reference plugin interface (`vocab_size`,
    `next_distributions(prefixes) -> float64 [n, V]`, pkg/src/speckit/models.py:32-63
    -- e.g. the reference's own MarkovModel / NgramModel / resolve_model outputs or
    a user plugin) through `HostRowsModel`, which uploads the rows it returns to
    HBM so the same GPU tree / warp / walk kernels consume them."""
    if hasattr(model, "tree_session") and hasattr(model, "tree_rows"):
        return model
    if hasattr(model, "next_distributions") and hasattr(model, "vocab_size"):
        return HostRowsModel.wrap(model)
    raise TypeError(
        f"{type(model).__name__} is not a LanguageModel: it needs vocab_size and next_distributions(prefixes)"
    )


def _normalize_rows(table: np.ndarray) -> np.ndarray:
    """models.py:66-74 (validation + one-time normalisation)."""
    table = np.asarray(table, dtype=np.float64)
    sums = table.sum(axis=-1, keepdims=True)
    if np.any(table < 0) or np.any(sums <= 0):
        raise ValueError("probability table rows must be non-negative with positive mass")
    if np.max(np.abs(sums - 1.0)) <= 1e-9:
        return table.copy()
    return table / sums


class _WorkspaceCache:
    """Tree workspaces by (K, B, V, D), per host thread (independent generation
    runs, e.g. tensor-parallel ranks as threads, never share device state)."""

    MAX_IDLE_BYTES = 1 << 30

    def __init__(self):
        self._tls = threading.local()

    def get(self, budget: int, B: int, V: int, D: int) -> K.TreeWorkspace:
        cache = getattr(self._tls, "ws", None)
        if cache is None:
            cache = self._tls.ws = {}
        key = (budget, B, V, D)
        ws = cache.get(key)
        if ws is None:
            # bound the device memory parked in idle workspaces (budget sweeps
            # build one per K; at K >= 2048 each is gigabytes next to a 70B target)
            if len(cache) > 4 or sum(w.buf.numel() for w in cache.values()) > self.MAX_IDLE_BYTES:
                cache.clear()
            ws = K.TreeWorkspace(budget, B, V, D)
            cache[key] = ws
        return ws


_WS = _WorkspaceCache()


class _TableSession:
    def __init__(self, model: "MarkovModel", prefix: Prefix, params: BuilderParams):
        self.model = model
        self.ws = _WS.get(params.budget, params.batch_size, model.vocab_size, params.max_depth)
        self.ws.begin(root_slot=0)
        self.ctx0 = model._context_tensor(prefix)
        self.rows = torch.empty((params.batch_size, model.vocab_size), dtype=torch.float64, device=self.ws.device)

    def batch_rows(self) -> torch.Tensor:
        m = self.model
        return K.markov_rows(m.table_dev, m.order, self.ctx0, self.ws, None, 0, True, self.rows)

    def advance(self, ctl) -> None:
        pass

    def finish(self, tree) -> None:
        tree.ctx0 = self.ctx0


class _TableStochastic:
    """Level rows for SpecInfer's stochastic builder (exact tables)."""

    def __init__(self, model: "MarkovModel"):
        self.model = model

    def level_rows(self, tree, level: list[int]) -> torch.Tensor:
        return self.model.rows_for_prefixes([tree.full_prefix(n) for n in level])

    def finish(self, tree) -> None:
        pass


class MarkovModel(LanguageModel):
    """Order-k Markov chain over a dense table (models.py:100-151), table in HBM."""

    backend = "markov"

    def __init__(self, table: np.ndarray, order: int = 1, _stationary: bool = False) -> None:
        if order < 1 and not _stationary:
            raise ValueError(f"order must be >= 1, got {order}")
        table = _normalize_rows(table)
        vocab = table.shape[1]
        if table.shape[0] != vocab**order:
            raise ValueError(f"table has {table.shape[0]} rows, expected vocab**order = {vocab**order}")
        self.table = table
        self.order = order
        self.vocab_size = vocab
        self.table_dev = torch.as_tensor(table).to(_device())

    def _row_index(self, prefix: Prefix) -> int:
        if self.order == 0:
            return 0
        context = prefix[-self.order :]
        context = (0,) * (self.order - len(context)) + context
        idx = 0
        for t in context:
            idx = idx * self.vocab_size + t
        return idx

    def _context_tensor(self, prefix: Prefix) -> torch.Tensor:
        n = max(self.order, 1)
        ctx = (0,) * n + tuple(prefix)
        return torch.tensor(ctx[-n:], dtype=torch.int32).to(self.table_dev.device)

    def next_distributions(self, prefixes) -> np.ndarray:
        idx = [self._row_index(_check_prefix(p, self.vocab_size)) for p in prefixes]
        if not idx:
            return np.empty((0, self.vocab_size))
        sel = torch.tensor(idx, dtype=torch.long, device=self.table_dev.device)
        return self.table_dev.index_select(0, sel).cpu().numpy()

    def power_smoothed(self, power: float) -> "MarkovModel":
        return type(self)._from_table(self.table**power, self.order)

    @classmethod
    def _from_table(cls, table, order):
        return MarkovModel(table, order=order)

    def to_json(self) -> str:
        return json.dumps({"backend": self.backend, "vocab_size": self.vocab_size, "order": self.order,
                           "table": self.table.tolist()})

    # ---- device-model protocol ----
    def tree_session(self, prefix: Prefix, params: BuilderParams) -> _TableSession:
        _check_prefix(prefix, self.vocab_size)
        return _TableSession(self, prefix, params)

    def rows_for_prefixes(self, prefixes) -> torch.Tensor:
        """fp64 rows [n, V] on the device for arbitrary prefixes (a gather of table rows)."""
        idx = [self._row_index(tuple(p)) for p in prefixes]
        sel = torch.tensor(idx, dtype=torch.long).to(self.table_dev.device, non_blocking=True)
        return self.table_dev.index_select(0, sel)

    def stochastic_session(self, prefix: Prefix, max_nodes: int, max_depth: int) -> "_TableStochastic":
        _check_prefix(prefix, self.vocab_size)
        return _TableStochastic(self)

    def tree_rows(self, tree) -> torch.Tensor:
        """Rows for the anchor and every node of a tree (GPU-built, or host-built
        like SpecInfer's stochastic trees)."""
        if tree.workspace is None:
            return self.rows_for_prefixes([tree.prefix] + [tree.full_prefix(nd.node_id) for nd in tree.nodes])
        n = len(tree)
        ws = tree.workspace
        ids = torch.arange(-1, n, dtype=torch.int32, device=ws.device)
        out = torch.empty((n + 1, self.vocab_size), dtype=torch.float64, device=ws.device)
        ctx0 = self._context_tensor(tree.prefix)
        return K.markov_rows(self.table_dev, self.order, ctx0, ws, ids, n + 1, False, out)

    def prefix_rows(self, prefix: Prefix) -> torch.Tensor:
        idx = self._row_index(_check_prefix(prefix, self.vocab_size))
        return self.table_dev[idx : idx + 1]


class TabularModel(MarkovModel):
    """Stationary backend: one fixed row (models.py:77-97) = an order-0 table."""

    backend = "tabular"

    def __init__(self, row: Sequence[float]) -> None:
        r = _normalize_rows(np.asarray(row, dtype=np.float64)[None, :])[0]
        super().__init__(r[None, :], order=0, _stationary=True)
        self.row = r

    def power_smoothed(self, power: float) -> "TabularModel":
        return TabularModel(self.row**power)

    def to_json(self) -> str:
        return json.dumps({"backend": self.backend, "vocab_size": self.vocab_size, "row": self.row.tolist()})


def make_synthetic(seed: int, vocab_size: int, sharpness: float, order: int = 1) -> MarkovModel:
    """Random Markov model with Dirichlet rows (models.py:265-279); same draws as the reference."""
    if vocab_size < 2:
        raise ValueError(f"vocab_size must be >= 2, got {vocab_size}")
    if sharpness <= 0:
        raise ValueError(f"sharpness must be > 0, got {sharpness}")
    gen = np.random.default_rng(seed)
    table = gen.dirichlet(np.full(vocab_size, sharpness), size=vocab_size**order)
    return MarkovModel(table, order=order)


def model_from_json(document: str) -> LanguageModel:
    data = json.loads(document)
    backend = data.get("backend")
    if backend == "tabular":
        return TabularModel(data["row"])
    if backend == "markov":
        return MarkovModel(np.asarray(data["table"]), order=data["order"])
    raise ValueError(f"unknown backend {backend!r}")


# ---------------------------------------------------------------------------
# host-row plugins (the drop-in boundary for models this package did not build)
# ---------------------------------------------------------------------------


def _host_rows(model, prefixes: list[Prefix]) -> np.ndarray:
    """`next_distributions` of a host plugin as a float64 [n, V] array (ValueError
    on a wrong shape -- the reference's contract, models.py:47-52)."""
    V = int(model.vocab_size)
    if not prefixes:
        return np.empty((0, V))
    rows = np.asarray(model.next_distributions(prefixes), dtype=np.float64)
    if rows.shape != (len(prefixes), V):
        raise ValueError(f"next_distributions returned shape {rows.shape}, expected {(len(prefixes), V)}")
    return np.ascontiguousarray(rows)


class _HostRowsSession:
    """Feeds the GPU tree builder from a host plugin: per round the batch's node
    paths are rebuilt from the workspace's ancestor-slot lists (each expanded
    node owns one slot, tree.cu tree_update_kernel), the plugin evaluates their
    full prefixes, and the float64 rows go up to HBM for sx_tree_round."""

    def __init__(self, adapter: "HostRowsModel", prefix: Prefix, params: BuilderParams):
        self.a = adapter
        self.prefix = prefix
        self.ws = _WS.get(params.budget, params.batch_size, adapter.vocab_size, params.max_depth)
        self.ws.begin(root_slot=0, pad_slot=0)
        self.slot_path: dict[int, Prefix] = {0: ()}
        self.first = True
        self.batch_n = 1

    def batch_rows(self) -> torch.Tensor:
        if self.first:
            self.first = False
            return self.a._upload(_host_rows(self.a.model, [self.prefix]))
        ws, n = self.ws, self.batch_n
        anc = ws.batch_anc()[:n].cpu().tolist()
        alen = ws.batch_anc_len()[:n].cpu().tolist()
        toks = ws.batch_tokens()[:n].cpu().tolist()
        slots = ws.batch_slots()[:n].cpu().tolist()
        K.IO["d2h"] += 4 * n * (len(anc[0]) + 3) if n else 0
        paths = []
        for b in range(n):
            path = self.slot_path[anc[b][alen[b] - 2]] + (toks[b],)
            self.slot_path[slots[b]] = path
            paths.append(self.prefix + path)
        return self.a._upload(_host_rows(self.a.model, paths))

    def advance(self, ctl) -> None:
        self.batch_n = ctl["batch_n"]

    def finish(self, tree) -> None:
        pass


class _HostRowsStochastic:
    """Level rows for the host-built trees (SpecInfer's stochastic builder, beam search)."""

    def __init__(self, adapter: "HostRowsModel"):
        self.a = adapter

    def level_rows(self, tree, level: list[int]) -> torch.Tensor:
        return self.a._upload(_host_rows(self.a.model, [tree.full_prefix(n) for n in level]))

    def finish(self, tree) -> None:
        pass


class HostRowsModel(LanguageModel):
    """Adapter for any reference-API LanguageModel plugin that is not one of this
    package's device models. Only the model rows come from the plugin (the
    reference contract: pure, batch-consistent float64 rows); tree building,
    scoring warps, the target-row cache and the acceptance walk run in the same
    sm_100a kernels as for device models. Rows are uploaded per draft round /
    per target pass (pinned staging, one H2D copy each)."""

    _cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
    _lock = threading.Lock()

    def __init__(self, model) -> None:
        self.model = model
        self.vocab_size = int(model.vocab_size)
        self.backend = f"host:{getattr(model, 'backend', type(model).__name__)}"
        self.device = _device()
        self._stage: torch.Tensor | None = None

    @classmethod
    def wrap(cls, model) -> "HostRowsModel":
        try:
            with cls._lock:
                a = cls._cache.get(model)
                if a is None:
                    a = cls._cache[model] = cls(model)
            return a
        except TypeError:  # not weak-referenceable: a fresh (stateless) adapter
            return cls(model)

    def _upload(self, rows: np.ndarray) -> torch.Tensor:
        n = rows.shape[0]
        need = rows.size
        if self._stage is None or self._stage.numel() < need:
            self._stage = torch.empty(max(need, 1), dtype=torch.float64).pin_memory()
        st = self._stage[:need]
        # the previous upload out of this staging buffer must have landed first
        torch.cuda.current_stream().synchronize()
        st.numpy()[:] = rows.reshape(-1)
        out = torch.empty((n, self.vocab_size), dtype=torch.float64, device=self.device)
        out.view(-1).copy_(st, non_blocking=True)
        K.IO["h2d"] += rows.nbytes
        return out

    # reference plugin API: the wrapped model's rows, unchanged
    def next_distributions(self, prefixes) -> np.ndarray:
        return _host_rows(self.model, [_check_prefix(p, self.vocab_size) for p in prefixes])

    def to_json(self) -> str:
        return self.model.to_json()

    # device-model protocol
    def tree_session(self, prefix: Prefix, params: BuilderParams) -> _HostRowsSession:
        return _HostRowsSession(self, _check_prefix(prefix, self.vocab_size), params)

    def stochastic_session(self, prefix: Prefix, max_nodes: int, max_depth: int) -> _HostRowsStochastic:
        _check_prefix(prefix, self.vocab_size)
        return _HostRowsStochastic(self)

    def tree_rows(self, tree) -> torch.Tensor:
        prefixes = [tree.prefix] + [tree.full_prefix(i) for i in range(len(tree))]
        return self._upload(_host_rows(self.model, prefixes))

    def prefix_rows(self, prefix: Prefix) -> torch.Tensor:
        return self._upload(_host_rows(self.model, [_check_prefix(prefix, self.vocab_size)]))
