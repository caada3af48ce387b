"""Thin torch-facing wrappers over the C ABI (device memory and streams only).

PyTorch allocates and owns every buffer; these functions pass raw pointers and
sizes to ``libspecexec_b200.so``. Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

import torch

from . import _lib
from ._lib import EPI_ADD_F32, EPI_BF16, EPI_F32, EPI_SWIGLU_BF16, EPI_SWIGLU_IL, call, ptr, stream_ptr

__all__ = [
    "EPI_ADD_F32",
    "EPI_BF16",
    "EPI_F32",
    "EPI_SWIGLU_BF16",
    "EPI_SWIGLU_IL",
    "gemm",
    "gemm_plan",
]

_ws_cache: dict[tuple[int, int], torch.Tensor] = {}

# host<->device bytes moved by the engine's control path (bench.py's e2e accounting)
IO = {"h2d": 0, "d2h": 0}
# kernels of this library launched by CUDA-graph replays (sx_launch_count sees only the capture)
GRAPH_KERNELS = [0]


class GemmProfiler:
    """Brackets every GEMM launch with CUDA events on the launching stream
    (bench.py: achieved FLOP/s of the dominant kernel over the timed region)."""

    def __init__(self):
        self.rec: list[tuple[int, int, int, int, torch.cuda.Event, torch.cuda.Event]] = []
        self._pool: list[torch.cuda.Event] = []

    def event(self) -> torch.cuda.Event:
        return self._pool.pop() if self._pool else torch.cuda.Event(enable_timing=True)

    def summary(self, min_m: int = 0) -> dict:
        torch.cuda.synchronize()
        flops = 0.0
        ms = 0.0
        n = 0
        for M, N, K, dual, e0, e1 in self.rec:
            if M < min_m:
                continue
            flops += 2.0 * M * N * K * (2 if dual else 1)
            ms += e0.elapsed_time(e1)
            n += 1
        return {"launches": n, "flops": flops, "ms": ms}

    def by_shape(self, top: int = 12, steps: int = 1) -> list[dict]:
        """Per (M, N, K, dual) shape: launches, ms and TFLOP/s (per step)."""
        torch.cuda.synchronize()
        agg: dict[tuple, list] = {}
        for M, N, K, dual, e0, e1 in self.rec:
            a = agg.setdefault((M, N, K, dual), [0, 0.0])
            a[0] += 1
            a[1] += e0.elapsed_time(e1)
        rows = []
        for (M, N, K, dual), (n, ms) in agg.items():
            fl = 2.0 * M * N * K * (2 if dual else 1) * n
            rows.append({"M": M, "N": N, "K": K, "dual": bool(dual), "launches_per_step": n / steps,
                         "ms_per_step": ms / steps, "tflops": fl / (ms / 1e3) / 1e12 if ms > 0 else 0.0})
        rows.sort(key=lambda r: -r["ms_per_step"])
        return rows[:top]


PROFILER: GemmProfiler | None = None


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tensor must live on a CUDA device")


def gemm_plan(M: int, N: int, K: int, dual: bool = False, splits: int = 0) -> tuple[int, int, int]:
    bn, sp, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong()
    _lib.check(
        _lib.load().sx_gemm_plan(M, N, K, int(dual), splits, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)),
        "sx_gemm_plan",
    )
    return bn.value, sp.value, ws.value


def _workspace(n_floats: int, device: torch.device) -> torch.Tensor | None:
    if n_floats <= 0:
        return None
    # per device AND host thread: stream-K flags / partials must not be shared by
    # GEMMs running concurrently on different streams (tensor-parallel thread-ranks)
    key = (device.index or 0, threading.get_ident())
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < n_floats:
        if ws is not None:
            _keep_alive.append(ws)  # captured CUDA graphs may still point at it
        # zero-filled: its prefix holds the stream-K partial-ready flags
        ws = torch.zeros(max(n_floats, 1 << 22), dtype=torch.float32, device=device)
        _ws_cache[key] = ws
    return ws


_keep_alive: list[torch.Tensor] = []


def gemm(
    x: torch.Tensor,
    w: torch.Tensor,
    out: torch.Tensor | None = None,
    epi: int = EPI_BF16,
    w2: torch.Tensor | None = None,
    splits: int = 0,
) -> torch.Tensor:
    """out[t, f] (op)= x[t, :] . w[f, :] on tcgen05 (bf16 in, fp32 accumulate)."""
    _require_cuda(x, w, w2)
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise ValueError("gemm: x and w must be bf16")
    if not x.is_contiguous() or not w.is_contiguous():
        raise ValueError("gemm: x and w must be contiguous")
    M, K = x.shape
    N = w.shape[0]
    if w.shape[1] != K:
        raise ValueError(f"gemm: inner dims differ ({K} vs {w.shape[1]})")
    if out is None:
        dt = torch.float32 if epi in (EPI_F32, EPI_ADD_F32) else torch.bfloat16
        ncol = N // 2 if epi == EPI_SWIGLU_IL else N
        out = (torch.zeros if epi == EPI_ADD_F32 else torch.empty)((M, ncol), dtype=dt, device=x.device)
    _, _, ws_need = gemm_plan(M, N, K, w2 is not None, splits)
    ws = _workspace(ws_need, x.device)
    prof = PROFILER
    if prof is not None and torch.cuda.is_current_stream_capturing():
        prof = None  # launches captured into a CUDA graph are not timed individually
    if prof is not None:
        e0 = prof.event()
        e0.record()
    call(
        "sx_gemm_bf16",
        ptr(w),
        ptr(w2),
        ptr(x),
        ptr(out),
        ptr(ws),
        ws.numel() if ws is not None else 0,
        M,
        N,
        K,
        out.stride(0),
        epi,
        splits,
        stream_ptr(),
    )
    if prof is not None:
        e1 = prof.event()
        e1.record()
        prof.rec.append((M, N, K, int(w2 is not None), e0, e1))
    return out


# ---------------------------------------------------------------------------
# canonical row kernels (sampling.py / engine.py semantics)
# ---------------------------------------------------------------------------

from ._lib import ROWS_ARGMAX_PACKED, ROWS_LOGITS_F32, ROWS_PROBS_F64, SCORE_ARGMAX, SCORE_RAW, SCORE_WARP  # noqa: E402

_scratch_cache: dict[tuple[int, str, int], torch.Tensor] = {}


def gemm_qkv_rope(x: torch.Tensor, w: torch.Tensor, H: int, KVH: int, pos, pos_base: int, slot, slot_base: int,
                  cos: torch.Tensor, sin: torch.Tensor, q: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor,
                  slots: int, splits: int = 0) -> None:
    """QKV projection whose epilogue applies RoPE and scatters K / V into the
    cache (sx_gemm_qkv_rope): q [M, H, 128] and the cache rows are written
    directly from the fp32 accumulators."""
    _require_cuda(x, w, q, kc, vc)
    M, Kd = x.shape
    N = w.shape[0]
    if N != (H + 2 * KVH) * 128:
        raise ValueError(f"gemm_qkv_rope: weight rows {N} != (H + 2 KVH) * 128")
    _, _, ws_need = gemm_plan(M, N, Kd, False, splits)
    ws = _workspace(ws_need, x.device)
    prof = PROFILER
    if prof is not None and torch.cuda.is_current_stream_capturing():
        prof = None
    if prof is not None:
        e0 = prof.event()
        e0.record()
    call("sx_gemm_qkv_rope", ptr(w), ptr(x), ptr(ws), ws.numel() if ws is not None else 0, M, H, KVH, Kd, ptr(pos),
         pos_base, ptr(slot), slot_base, ptr(cos), ptr(sin), ptr(q), ptr(kc), ptr(vc), slots, splits, stream_ptr())
    if prof is not None:
        e1 = prof.event()
        e1.record()
        prof.rec.append((M, N, Kd, 0, e0, e1))


def gemm_rs(x: torch.Tensor, w: torch.Tensor, peer_inbox: torch.Tensor, rank: int, world: int, splits: int = 0) -> None:
    """Row-parallel projection fused with the reduce-scatter half of its
    all-reduce (sx_gemm_bf16_rs): the epilogue writes each feature slice of
    this rank's bf16 partial into its owner's inbox (peer_inbox: device int64
    pointer table)."""
    _require_cuda(x, w, peer_inbox)
    M, Kd = x.shape
    N = w.shape[0]
    _, _, ws_need = gemm_plan(M, N, Kd, False, splits)
    ws = _workspace(ws_need, x.device)
    call("sx_gemm_bf16_rs", ptr(w), ptr(x), ptr(peer_inbox), rank, world, ptr(ws), ws.numel() if ws is not None else 0,
         M, N, Kd, splits, stream_ptr())


def scratch(nbytes: int, device: torch.device, tag: str, zero: bool = False) -> torch.Tensor:
    """Per (device, tag, host thread) scratch buffer, grown on demand; `zero`:
    zero-filled when (re)allocated (kernels that keep counters in it reset them
    themselves after each launch)."""
    key = (device.index or 0, tag, threading.get_ident())
    buf = _scratch_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            _keep_alive.append(buf)
        buf = (torch.zeros if zero else torch.empty)(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
        _scratch_cache[key] = buf
    return buf


def row_kind(rows: torch.Tensor) -> int:
    if rows.dtype == torch.float32:
        return ROWS_LOGITS_F32
    if rows.dtype == torch.float64:
        return ROWS_PROBS_F64
    if rows.dtype == torch.int64:
        return ROWS_ARGMAX_PACKED
    raise ValueError(f"rows must be fp32 logits, fp64 probabilities or int64 argmax keys, got {rows.dtype}")


def warp_rows(rows: torch.Tensor, temperature: float, top_p: float, row_ids: torch.Tensor | None = None) -> torch.Tensor:
    """apply_warp of each row (fp32 logits or fp64 probabilities) -> fp64 rows."""
    _require_cuda(rows)
    if rows.stride(-1) != 1:
        rows = rows.contiguous()
    n = rows.shape[0] if row_ids is None else row_ids.numel()
    V = rows.shape[1]
    out = torch.empty((n, V), dtype=torch.float64, device=rows.device)
    lib = _lib.load()
    sc = scratch(lib.sx_warp_scratch_bytes(n, V), rows.device, "warp")
    call("sx_warp_rows", ptr(rows), row_kind(rows), rows.stride(0), V, ptr(row_ids), n, float(temperature), float(top_p),
         ptr(out), V, ptr(sc), stream_ptr())
    return out


def sample_rows(warped: torch.Tensor, uniforms) -> torch.Tensor:
    _require_cuda(warped)
    n, V = warped.shape
    u = torch.as_tensor(np.asarray(uniforms, dtype=np.float64)).to(warped.device)
    out = torch.empty(n, dtype=torch.int32, device=warped.device)
    call("sx_sample_rows", ptr(warped), warped.stride(0), V, ptr(u), n, ptr(out), stream_ptr())
    return out.cpu()


def softmax_rows(logits: torch.Tensor, row_ids: torch.Tensor | None = None) -> torch.Tensor:
    """Canonical float64 probabilities of fp32 logits rows."""
    _require_cuda(logits)
    n = logits.shape[0] if row_ids is None else row_ids.numel()
    V = logits.shape[1]
    out = torch.empty((n, V), dtype=torch.float64, device=logits.device)
    call("sx_softmax_rows", ptr(logits), logits.stride(0), V, ptr(row_ids), n, ptr(out), V, stream_ptr())
    return out


def rows_argmax_packed(logits: torch.Tensor, v0: int, out: torch.Tensor) -> torch.Tensor:
    """KV1: int64 key per row of a vocab slice (columns v0 .. v0 + Vl) whose MAX
    over the slices is the global argmax (lowest id on ties); out [n, 1] int64."""
    _require_cuda(logits)
    n, Vl = logits.shape
    call("sx_rows_argmax_packed", ptr(logits), logits.stride(0), n, Vl, v0, ptr(out), stream_ptr())
    return out


def argmax_rows(rows: torch.Tensor) -> torch.Tensor:
    _require_cuda(rows)
    n, V = rows.shape
    out = torch.empty(n, dtype=torch.int32, device=rows.device)
    call("sx_argmax_rows", ptr(rows), row_kind(rows), rows.stride(0), V, n, ptr(out), stream_ptr())
    return out


class WalkResult:
    __slots__ = ("tokens", "fell_off", "cursor", "path_rows")

    def __init__(self, tokens, fell_off, cursor, path_rows):
        self.tokens = tokens
        self.fell_off = fell_off
        self.cursor = cursor
        self.path_rows = path_rows


def verify_walk(rows: torch.Tensor, parent: torch.Tensor, token: torch.Tensor, n_nodes: int, start_cursor: int,
                uniforms: np.ndarray, max_steps: int, temperature: float, top_p: float,
                out_host: torch.Tensor | None = None) -> WalkResult:
    """Acceptance walk over cached target rows (engine.py:118-128) on one CTA."""
    dev = rows.device
    V = rows.shape[1]  # 1 for int64 argmax keys (KV1): the walk reads only the key
    lib = _lib.load()
    sc = scratch(lib.sx_row_scratch_bytes(V), dev, "walk")
    u = torch.as_tensor(np.ascontiguousarray(uniforms[:max_steps], dtype=np.float64))
    if u.numel() < max_steps:
        u = torch.cat([u, torch.zeros(max_steps - u.numel(), dtype=torch.float64)])
    u = u.to(dev, non_blocking=True)
    out = torch.empty(3 + 2 * max_steps, dtype=torch.int32, device=dev)
    call("sx_verify_walk", ptr(rows), row_kind(rows), rows.stride(0), V, ptr(parent), ptr(token), n_nodes,
         start_cursor, ptr(u), max_steps, float(temperature), float(top_p), ptr(out), ptr(sc), stream_ptr())
    if out_host is None:
        host = out.cpu()
    else:
        host = out_host[: out.numel()]
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    IO["h2d"] += 8 * max_steps
    IO["d2h"] += 4 * out.numel()
    h = host.tolist()
    n = h[0]
    return WalkResult(h[3 : 3 + n], bool(h[1]), h[2], h[3 + max_steps : 3 + max_steps + n - (1 if h[1] else 0)])


# ---------------------------------------------------------------------------
# stage-1 tree workspace
# ---------------------------------------------------------------------------

_OFF_NAMES = ["ctl", "b_node", "b_nll", "b_depth", "b_lex", "b_slot", "b_token", "b_anc", "b_anc_len",
              "f_anc", "f_anc_len", "f_depth", "f_token", "w_rows", "b_pos", "b_dense", "total", "r_aux"]


class TreeWorkspace:
    """Device state of one draft-tree build (csrc/tree_layout.h)."""

    def __init__(self, K: int, B: int, V: int, D: int, device: torch.device | None = None):
        lib = _lib.load()
        self.K, self.B, self.V, self.D = K, B, V, D
        nbytes = lib.sx_tree_workspace_bytes(K, B, V, D)
        if nbytes < 0:
            raise ValueError("invalid tree parameters")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        offs = (ctypes.c_longlong * len(_OFF_NAMES))()
        lib.sx_tree_offsets(K, B, V, D, offs, len(_OFF_NAMES))
        self.off = dict(zip(_OFF_NAMES, list(offs)))
        self.ctl_host = torch.zeros(16, dtype=torch.int32).pin_memory()
        self.cap = lib.sx_tree_survivor_cap(K, B, V, D)
        self.last_round = None
        self.overflow_retries = 0
        self.rounds = 0
        # pinned staging of the finished tree (parent, token, slot | edge): copied
        # asynchronously so the host builds DraftTree while the target pass runs
        self.host_i = torch.zeros((3, K + 1), dtype=torch.int32).pin_memory()
        self.host_e = torch.zeros(K + 1, dtype=torch.float64).pin_memory()
        self.host_ready = torch.cuda.Event()
        self.pending_tree = None

    def view(self, name: str, dtype: torch.dtype, n: int) -> torch.Tensor:
        o = self.off[name]
        item = torch.empty((), dtype=dtype).element_size()
        return self.buf[o : o + n * item].view(dtype)

    # batch inputs of the next draft call
    def batch_tokens(self) -> torch.Tensor:
        return self.view("b_token", torch.int32, self.B)

    def batch_depth(self) -> torch.Tensor:
        return self.view("b_depth", torch.int32, self.B)

    def batch_slots(self) -> torch.Tensor:
        return self.view("b_slot", torch.int32, self.B)

    def batch_anc(self) -> torch.Tensor:
        return self.view("b_anc", torch.int32, self.B * (self.D + 1)).view(self.B, self.D + 1)

    def batch_anc_len(self) -> torch.Tensor:
        return self.view("b_anc_len", torch.int32, self.B)

    def final_tables(self, n_rows: int):
        anc = self.view("f_anc", torch.int32, (self.K + 1) * (self.D + 1)).view(self.K + 1, self.D + 1)[:n_rows]
        return (anc, self.view("f_anc_len", torch.int32, self.K + 1)[:n_rows],
                self.view("f_depth", torch.int32, self.K + 1)[:n_rows], self.view("f_token", torch.int32, self.K + 1)[:n_rows])

    def batch_dense(self) -> torch.Tensor:
        return self.view("b_dense", torch.int32, self.B)

    def begin(self, root_slot: int = 0, pad_slot: int = 0) -> None:
        if _lib.load().sx_tree_survivor_cap(self.K, self.B, self.V, self.D) != self.cap:
            raise RuntimeError("tree workspace laid out under another survivor capacity (sx_tree_set_survivor_cap)")
        self.rounds = 0
        call("sx_tree_begin", ptr(self.buf), self.K, self.B, self.V, self.D, root_slot, pad_slot, stream_ptr())

    def launch_round(self, rows: torch.Tensor, score_mode: int, temperature: float = 1.0, top_p: float = 1.0) -> None:
        """Enqueue scoring + update + control-block readback (capturable in a CUDA graph)."""
        _require_cuda(rows)
        self.last_round = (rows, score_mode, temperature, top_p)
        call("sx_tree_round", ptr(self.buf), self.K, self.B, self.V, self.D, ptr(rows), row_kind(rows), rows.stride(0),
             score_mode, float(temperature), float(top_p), self.ctl_host.data_ptr(), stream_ptr())

    def _retry_sliced(self) -> list:
        """The last round overflowed the survivor buffer (nothing was committed):
        re-run the same rows in slices whose candidates fit, merging each slice
        into the K best (sx_tree_round_rows; the last slice picks the next batch)."""
        rows, mode, temp, top_p = self.last_round
        batch_n = self.ctl_host.tolist()[5]
        per = max(1, int(self.cap // self.V))
        call("sx_tree_clear_overflow", ptr(self.buf), self.K, self.B, self.V, self.D, stream_ptr())
        self.overflow_retries += 1
        for r0 in range(0, batch_n, per):
            r1 = min(batch_n, r0 + per)
            call("sx_tree_round_rows", ptr(self.buf), self.K, self.B, self.V, self.D, ptr(rows), row_kind(rows),
                 rows.stride(0), mode, float(temp), float(top_p), r0, r1, int(r1 == batch_n),
                 self.ctl_host.data_ptr(), stream_ptr())
            torch.cuda.current_stream().synchronize()
            c = self.ctl_host.tolist()
            if c[8]:
                raise RuntimeError(f"tree: survivor overflow in a {r1 - r0}-row slice (cap {self.cap})")
        return c

    def round(self, rows: torch.Tensor, score_mode: int, temperature: float = 1.0, top_p: float = 1.0) -> dict:
        """Score the current batch's rows, update the tree; returns the control block."""
        self.launch_round(rows, score_mode, temperature, top_p)
        return self.read_ctl()

    def read_ctl(self) -> dict:
        IO["d2h"] += 56
        torch.cuda.current_stream().synchronize()
        self.rounds += 1
        c = self.ctl_host.tolist()
        if c[8]:
            c = self._retry_sliced()
        return {"count": c[1], "has_thr": c[2], "slot_next": c[4], "batch_n": c[5]}

    def batch_pos(self) -> torch.Tensor:
        return self.view("b_pos", torch.int32, self.B)

    def finalize(self, n: int, root_token: int = 0):
        parent = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        token = torch.empty_like(parent)
        depth = torch.empty_like(parent)
        slot = torch.empty_like(parent)
        edge = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)
        call("sx_tree_finalize", ptr(self.buf), self.K, self.B, self.V, self.D, int(root_token), ptr(parent), ptr(token),
             ptr(edge), ptr(depth), ptr(slot), stream_ptr())
        return parent[:n], token[:n], edge[:n], depth[:n], slot[:n]

    def stage_to_host(self, parent, token, slot, edge) -> None:
        """Async D2H of the finished tree into the pinned staging buffers."""
        n = parent.numel()
        self.host_i[0, :n].copy_(parent, non_blocking=True)
        self.host_i[1, :n].copy_(token, non_blocking=True)
        self.host_i[2, :n].copy_(slot, non_blocking=True)
        self.host_e[:n].copy_(edge, non_blocking=True)
        self.host_ready.record()
        IO["d2h"] += 20 * n


def markov_rows(table: torch.Tensor, order: int, ctx0: torch.Tensor, ws: TreeWorkspace, node_ids: torch.Tensor | None,
                n_nodes: int, from_batch: bool, out: torch.Tensor) -> torch.Tensor:
    V = table.shape[1]
    call("sx_markov_rows", ptr(table), V, order, ptr(ctx0), ptr(ws.buf), ws.K, ws.B, ws.D, ptr(node_ids), n_nodes,
         int(from_batch), ptr(out), out.stride(0), stream_ptr())
    return out
