"""Thin torch-facing wrappers over the C ABI (device memory and streams only).

PyTorch allocates and owns every buffer; these functions pass raw pointers and
sizes to ``libspecexec_b200.so``. Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import EPI_ADD_F32, EPI_BF16, EPI_F32, EPI_SWIGLU_BF16, call, ptr, stream_ptr

__all__ = [
    "EPI_ADD_F32",
    "EPI_BF16",
    "EPI_F32",
    "EPI_SWIGLU_BF16",
    "gemm",
    "gemm_plan",
]

_ws_cache: dict[tuple[int, int], torch.Tensor] = {}


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
    key = (device.index or 0, 0)
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < n_floats:
        ws = torch.empty(max(n_floats, 1 << 20), dtype=torch.float32, device=device)
        _ws_cache[key] = ws
    return ws


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
        out = (torch.zeros if epi == EPI_ADD_F32 else torch.empty)((M, N), dtype=dt, device=x.device)
    _, _, ws_need = gemm_plan(M, N, K, w2 is not None, splits)
    ws = _workspace(ws_need, x.device)
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
    return out
