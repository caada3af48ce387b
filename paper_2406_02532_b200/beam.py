"""Beam-search draft trees on the GPU (build_beam, pkg/src/speckit/tree.py:330-380;
the paper's Appendix F ablation).

Per step: ONE draft forward over the current beams (the device model's level
rows, the same path SpecInfer's stochastic builder uses), the scored rows
(canonical warp or raw probabilities) on the device, and `sx_beam_step`: every
row's candidates sorted by (nll, token) with the canonical log, the best
`beam_size` per row, then the global best `beam_size` by (nll, path) in one
CTA. Only the kept candidates (<= beam_size of them) come back to the host,
which keeps the paths and finally emits the prefix closure of the last beam
with node ids in (length, path) order, exactly like the reference.
"""

from __future__ import annotations

import torch

from . import _lib
from . import kernels as K
from .models import as_device_model
from .sampling import SamplingConfig
from .specinfer import _scored_rows
from .tree import ROOT, DraftTree

Prefix = tuple[int, ...]


def build_beam(prefix, draft, beam_size: int, max_len: int, warp: SamplingConfig | None = None,
               warp_scores: bool = True) -> DraftTree:
    """Standard beam search; the tree is the prefix closure of the final beam."""
    if beam_size < 1:
        raise ValueError(f"beam_size must be >= 1, got {beam_size}")
    if max_len < 1:
        raise ValueError(f"max_len must be >= 1, got {max_len}")
    dm = as_device_model(draft)
    prefix = tuple(int(t) for t in prefix)
    V = dm.vocab_size
    session = dm.stochastic_session(prefix, beam_size * max_len, max_len)
    search = DraftTree(prefix)  # every kept hypothesis, for the model's KV / row bookkeeping
    dev = torch.device("cuda", torch.cuda.current_device())
    temp, top_p = (warp.temperature, warp.top_p) if (warp is not None and warp_scores) else (None, None)
    k = beam_size
    beams: list[tuple[float, Prefix, int]] = [(0.0, (), ROOT)]  # (nll, path, search node)
    edges: dict[Prefix, float] = {}
    rounds = 0
    for _ in range(max_len):
        nb = len(beams)
        rows = session.level_rows(search, [b[2] for b in beams])
        rounds += 1
        q = torch.empty((nb, V), dtype=torch.float64, device=dev)
        _scored_rows(rows, q, temp, top_p)
        order = sorted(range(nb), key=lambda i: beams[i][1])  # lex rank of the (equal-length) paths
        rank = [0] * nb
        for r, i in enumerate(order):
            rank[i] = r
        b_nll = torch.tensor([b[0] for b in beams], dtype=torch.float64).to(dev, non_blocking=True)
        b_rank = torch.tensor(rank, dtype=torch.int32).to(dev, non_blocking=True)
        c_nll = torch.empty(nb * k, dtype=torch.float64, device=dev)  # per-row candidates
        c_edge = torch.empty_like(c_nll)
        c_tok = torch.empty(nb * k, dtype=torch.int32, device=dev)
        c_cnt = torch.empty(nb, dtype=torch.int32, device=dev)
        out = torch.empty(1 + 2 * k, dtype=torch.int32, device=dev)  # n, beam[k], tok[k]
        o_f = torch.empty(2 * k, dtype=torch.float64, device=dev)  # nll[k], edge[k]
        scratch = K.scratch(_lib.load().sx_beam_scratch_bytes(nb, V), dev, "beam")
        _lib.call("sx_beam_step", _lib.ptr(q), V, V, nb, _lib.ptr(b_nll), _lib.ptr(b_rank), k, _lib.ptr(scratch),
                  _lib.ptr(c_nll), _lib.ptr(c_edge), _lib.ptr(c_tok), _lib.ptr(c_cnt), _lib.ptr(out[0:1]),
                  _lib.ptr(o_f[:k]), _lib.ptr(o_f[k:]), _lib.ptr(out[1 : 1 + k]), _lib.ptr(out[1 + k :]),
                  _lib.stream_ptr())
        oi, of = out.cpu().tolist(), o_f.cpu().tolist()
        K.IO["h2d"] += 12 * nb
        K.IO["d2h"] += 4 * len(oi) + 8 * len(of)
        n = oi[0]
        if n == 0:
            break
        kept = []
        for j in range(n):
            bi, tok, nll, edge = oi[1 + j], oi[1 + k + j], of[j], of[k + j]
            parent_node = beams[bi][2]
            node = search.add_child(parent_node, tok, edge)
            path = beams[bi][1] + (tok,)
            edges[path] = edge
            kept.append((nll, path, node))
        beams = kept
    session.finish(search)
    tree = DraftTree(prefix)
    tree.rounds = rounds
    keep: set[Prefix] = set()
    for _, path, _ in beams:
        for end in range(1, len(path) + 1):
            keep.add(path[:end])
    path_to_id: dict[Prefix, int] = {(): ROOT}
    for path in sorted(keep, key=lambda p: (len(p), p)):
        path_to_id[path] = tree.add_child(path_to_id[path[:-1]], path[-1], edges[path])
    return tree
