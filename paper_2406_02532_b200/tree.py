"""Draft trees and the GPU best-first (SSSP) builder.

Host-side data structures keep the reference API (pkg/src/speckit/tree.py):
`BuilderParams` (:36-55), `DraftNode` (:58-68), `FlattenedTree` (:71-82),
`DraftTree` (:85-205), `flatten` (:208-219). `build_sssp` (:240-327) runs on the
GPU: each round the draft model produces rows for the current batch *on the
device* and `sx_tree_round` (csrc/tree.cu) scores, selects and picks the next
batch; only the control block (batch size) crosses to the host per round.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from .sampling import SamplingConfig

ROOT = -1
Prefix = tuple[int, ...]


@dataclass(frozen=True)
class BuilderParams:
    """budget K (nodes, root excluded), max_depth D, batch_size B (tree.py:36-55)."""

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
    node_id: int
    parent: int
    token: int
    edge_logprob: float
    cum_logprob: float
    depth: int
    multiplicity: int = 1


@dataclass
class FlattenedTree:
    order: list[int]
    ancestor_mask: np.ndarray


class DraftTree:
    """Prefix-closed tree of draft tokens anchored at a prompt prefix (tree.py:85-205)."""

    def __init__(self, prefix: Prefix) -> None:
        self.prefix: Prefix = tuple(prefix)
        self._nodes: list[DraftNode] = []
        self._fill = None  # GPU-built trees: nodes materialise on first access
        self._n = 0
        self.rounds: int = 0
        self.draft_dists = None
        self._children: dict[int, list[int]] = {ROOT: []}
        # device-side copies filled by the GPU builder (parent/token per node id)
        self.device_parent = None
        self.device_token = None
        self.workspace = None

    @property
    def nodes(self) -> list[DraftNode]:
        if self._fill is not None:
            fill, self._fill = self._fill, None
            fill(self)
        return self._nodes

    def __len__(self) -> int:
        return self._n if self._fill is not None else len(self._nodes)

    def add_child(self, parent: int, token: int, edge_logprob: float) -> int:
        if parent != ROOT:
            self._check_id(parent)
        node_id = len(self.nodes)
        parent_cum = 0.0 if parent == ROOT else self.nodes[parent].cum_logprob
        parent_depth = 0 if parent == ROOT else self.nodes[parent].depth
        self.nodes.append(
            DraftNode(node_id, parent, int(token), float(edge_logprob), parent_cum + float(edge_logprob), parent_depth + 1)
        )
        self._children[node_id] = []
        self._children[parent].append(node_id)
        return node_id

    def _check_id(self, node_id: int) -> None:
        if not 0 <= node_id < len(self.nodes):
            raise KeyError(f"no node with id {node_id}")

    def children_of(self, node_id: int) -> list[int]:
        self.nodes  # noqa: B018  (materialise a GPU-built tree)
        if node_id != ROOT:
            self._check_id(node_id)
        return list(self._children[node_id])

    def child_with_token(self, node_id: int, token: int) -> int | None:
        self.nodes  # noqa: B018
        for child in self._children[node_id]:
            if self.nodes[child].token == token:
                return child
        return None

    def path_tokens(self, node_id: int) -> Prefix:
        if node_id == ROOT:
            return ()
        self._check_id(node_id)
        path = []
        while node_id != ROOT:
            node = self.nodes[node_id]
            path.append(node.token)
            node_id = node.parent
        return tuple(reversed(path))

    def full_prefix(self, node_id: int) -> Prefix:
        return self.prefix + self.path_tokens(node_id)

    def cumulative_logprob(self, node_id: int) -> float:
        self._check_id(node_id)
        total = 0.0
        while node_id != ROOT:
            node = self.nodes[node_id]
            total += node.edge_logprob
            node_id = node.parent
        return total

    def max_depth(self) -> int:
        return max((n.depth for n in self.nodes), default=0)

    def total_mass(self) -> float:
        masses = sorted(math.exp(n.cum_logprob) for n in self.nodes)
        return float(sum(masses))

    def to_json(self) -> str:
        return json.dumps(
            {
                "prefix": list(self.prefix),
                "nodes": [
                    {"id": n.node_id, "parent": n.parent, "token": n.token, "edge_logprob": n.edge_logprob,
                     "cum_logprob": n.cum_logprob}
                    for n in self.nodes
                ],
            }
        )

    @classmethod
    def from_json(cls, document: str) -> "DraftTree":
        data = json.loads(document)
        tree = cls(prefix=tuple(data["prefix"]))
        for record in data["nodes"]:
            node_id = tree.add_child(record["parent"], record["token"], record["edge_logprob"])
            if node_id != record["id"]:
                raise ValueError(f"node ids must be contiguous; got {record['id']}")
            if abs(tree.nodes[node_id].cum_logprob - record["cum_logprob"]) > 1e-9:
                raise ValueError(f"inconsistent cum_logprob for node {node_id}")
        return tree


def flatten(tree: DraftTree) -> FlattenedTree:
    """Parents-first order plus the dense ancestor mask (tree.py:208-219).

    The GPU engine never materialises this mask; attention uses per-row
    ancestor lists (csrc/attention.cu). Kept for API compatibility."""
    order = [n.node_id for n in tree.nodes]
    m = len(order) + 1
    mask = np.zeros((m, m), dtype=bool)
    mask[0, 0] = True
    for node in tree.nodes:
        pos = node.node_id + 1
        mask[pos] = mask[node.parent + 1]
        mask[pos, pos] = True
    return FlattenedTree(order=order, ancestor_mask=mask)


def score_mode(warp: SamplingConfig | None, warp_scores: bool) -> tuple[int, float, float]:
    """_scored_dist (tree.py:222-227): which scoring kernel the round uses."""
    from ._lib import SCORE_ARGMAX, SCORE_RAW, SCORE_WARP

    if warp is None or not warp_scores or warp.is_identity:
        return SCORE_RAW, 1.0, 1.0
    if warp.temperature == 0.0:
        return SCORE_ARGMAX, 0.0, 1.0
    return SCORE_WARP, float(warp.temperature), float(warp.top_p)


def tree_tables(tree: DraftTree) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """Host-built trees (e.g. SpecInfer's stochastic trees): the ancestor tables
    of the flattened tree (tree.py:208-219) in the layout the GPU builder's
    finalize produces -- per row (0 = root, i+1 = node i): ancestor rows
    root-first ending with itself [n+1, D+1], their count, depth and token."""
    n = len(tree.nodes)
    A = tree.max_depth() + 1
    anc = np.zeros((n + 1, A), dtype=np.int32)
    alen = np.ones(n + 1, dtype=np.int32)
    depth = np.zeros(n + 1, dtype=np.int32)
    tok = np.zeros(n + 1, dtype=np.int32)
    tok[0] = tree.prefix[-1] if tree.prefix else 0
    for nd in tree.nodes:  # parents have smaller ids
        r, pr = nd.node_id + 1, nd.parent + 1
        k = alen[pr]
        anc[r, :k] = anc[pr, :k]
        anc[r, k] = r
        alen[r] = k + 1
        depth[r] = nd.depth
        tok[r] = nd.token
    return anc, alen, depth, tok


def _tree_from_device(prefix: Prefix, ws, n: int, rounds: int) -> DraftTree:
    """DraftTree whose host nodes are built from the pinned staging buffers on
    first access (after the copies land): the target pass is already enqueued
    by then, so the host-side construction overlaps GPU work."""
    tree = DraftTree(prefix)
    tree.rounds = rounds
    tree._n = n

    def fill(t: DraftTree) -> None:
        ws.host_ready.synchronize()
        if ws.pending_tree is t:
            ws.pending_tree = None
        par, tok = ws.host_i[0, :n].tolist(), ws.host_i[1, :n].tolist()
        for p, k, e in zip(par, tok, ws.host_e[:n].tolist()):
            t.add_child(p, k, e)
        t.host_slot_staged = ws.host_i[2, :n].tolist()

    tree._fill = fill
    return tree


def build_sssp(
    prefix: Prefix,
    draft,
    params: BuilderParams,
    warp: SamplingConfig | None = None,
    warp_scores: bool = True,
) -> DraftTree:
    """Best-first search for the budget-many most likely continuations, on the GPU.

    Exactly the reference's top-`budget` sequences of length <= max_depth under
    (nll asc, depth asc, path-lex asc), with the same per-round batches (and so
    the same `rounds`) for the same batch_size.
    """
    from .models import as_device_model

    dm = as_device_model(draft)
    prefix = tuple(int(t) for t in prefix)
    session = dm.tree_session(prefix, params)
    mode, temp, top_p = score_mode(warp, warp_scores)
    ws = session.ws
    run_round = getattr(session, "run_round", None)
    while True:
        if run_round is not None:  # the session fuses draft forward + round (CUDA graph)
            ctl = run_round(mode, temp, top_p)
        else:
            rows = session.batch_rows()
            ctl = ws.round(rows, mode, temp, top_p)
        if ctl["batch_n"] == 0:
            break
        session.advance(ctl)
    n = ctl["count"]
    if ws.pending_tree is not None:  # the staging buffers are about to be reused
        ws.pending_tree.nodes  # noqa: B018  (materialise the previous tree first)
    parent, token, edge, depth, slot = ws.finalize(n, prefix[-1] if prefix else 0)
    ws.stage_to_host(parent, token, slot, edge)
    tree = _tree_from_device(prefix, ws, n, ws.rounds)
    ws.pending_tree = tree
    tree.device_parent, tree.device_token, tree.workspace = parent, token, ws
    tree.device_depth = depth
    tree.device_slot = slot
    session.finish(tree)
    return tree
