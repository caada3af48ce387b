"""ctypes binding of the in-tree C-ABI library ``libspecexec_b200.so``.

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every device call raises. The declarations mirror
``include/specexec_b200.h``.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
# SX_LIB_PATH: an instrumented build of the same library (e.g. `make TRACE=1` for
# tools/tree_round_bench.py --trace); the product default is the in-tree build
LIB_PATH = pathlib.Path(os.environ.get("SX_LIB_PATH", _HERE / "libspecexec_b200.so"))

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)
_llp = ctypes.POINTER(ctypes.c_longlong)

# name -> (restype, argtypes); must list every symbol the header declares.
SIGNATURES: dict[str, tuple] = {
    "sx_abi_version": (_c_int, []),
    "sx_last_error": (ctypes.c_char_p, []),
    "sx_launch_count": (_c_ll, []),
    "sx_gemm_set_pair_mode": (_c_int, [_c_int]),
    "sx_gemm_set_gemv": (_c_int, [_c_int]),
    "sx_gemm_plan": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _ip, _ip, _llp]),
    "sx_gemm_bf16": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_ll, _c_int, _c_int, _c_int, _c_ll, _c_int, _c_int, _vp],
    ),
    "sx_tree_workspace_bytes": (_c_ll, [_c_int, _c_int, _c_int, _c_int]),
    "sx_tree_offsets": (_c_int, [_c_int, _c_int, _c_int, _c_int, _llp, _c_int]),
    "sx_tree_begin": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp]),
    "sx_tree_round": (
        _c_int,
        [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_ll, _c_int, _c_dbl, _c_dbl, _vp, _vp],
    ),
    "sx_tree_set_impl": (_c_int, [_c_int]),
    "sx_tree_survivor_cap": (_c_ll, [_c_int, _c_int, _c_int, _c_int]),
    "sx_tree_set_survivor_cap": (_c_int, [_c_ll]),
    "sx_tree_clear_overflow": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "sx_tree_round_rows": (
        _c_int,
        [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_ll, _c_int, _c_dbl, _c_dbl, _c_int, _c_int, _c_int,
         _vp, _vp],
    ),
    "sx_tree_finalize": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sx_markov_rows": (
        _c_int,
        [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_ll, _vp],
    ),
    "sx_row_scratch_bytes": (_c_ll, [_c_int]),
    "sx_verify_walk": (
        _c_int,
        [_vp, _c_int, _c_ll, _c_int, _vp, _vp, _c_int, _c_int, _vp, _c_int, _c_dbl, _c_dbl, _vp, _vp, _vp],
    ),
    "sx_warp_scratch_bytes": (_c_ll, [_c_int, _c_int]),
    "sx_warp_rows": (
        _c_int,
        [_vp, _c_int, _c_ll, _c_int, _vp, _c_int, _c_dbl, _c_dbl, _vp, _c_ll, _vp, _vp],
    ),
    "sx_softmax_rows": (_c_int, [_vp, _c_ll, _c_int, _vp, _c_int, _vp, _c_ll, _vp]),
    "sx_argmax_rows": (_c_int, [_vp, _c_int, _c_ll, _c_int, _c_int, _vp, _vp]),
    "sx_rows_argmax_packed": (_c_int, [_vp, _c_ll, _c_int, _c_int, _c_int, _vp, _vp]),
    "sx_sample_rows": (_c_int, [_vp, _c_ll, _c_int, _vp, _c_int, _vp, _vp]),
    "sx_beam_scratch_bytes": (_c_ll, [_c_int, _c_int]),
    "sx_beam_step": (
        _c_int,
        [_vp, _c_ll, _c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "sx_sample_rows_idx": (_c_int, [_vp, _c_ll, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp]),
    "sx_specinfer_verify": (
        _c_int,
        [_vp, _c_int, _c_ll, _c_int, _vp, _c_ll, _vp, _vp, _vp, _vp, _vp, _c_int, _vp, _c_int, ctypes.c_double,
         ctypes.c_double, _vp, _vp, _vp],
    ),
    "sx_embed": (_c_int, [_vp, _vp, _c_int, _c_int, _vp, _vp]),
    "sx_rmsnorm": (_c_int, [_vp, _vp, _c_int, _c_int, ctypes.c_float, _vp, _vp]),
    "sx_add_rmsnorm": (_c_int, [_vp, _vp, _c_int, _vp, _c_int, _c_int, ctypes.c_float, _vp, _vp]),
    "sx_gemm_bf16_rs": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _vp, _c_ll, _c_int, _c_int, _c_int, _c_int, _vp]),
    "sx_gemm_qkv_rope": (
        _c_int,
        [_vp, _vp, _vp, _c_ll, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp,
         _c_ll, _c_int, _vp],
    ),
    "sx_tp_reduce_bcast": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp]),
    "sx_rope_kv": (
        _c_int,
        [_vp, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _c_ll, _vp],
    ),
    "sx_tree_attention": (
        _c_int,
        [_vp, _vp, _vp, _c_ll, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp],
    ),
    "sx_tree_attention_ws": (
        _c_int,
        [_vp, _vp, _vp, _c_ll, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp, _c_ll, _vp],
    ),
    "sx_tree_attention_ws_bytes": (_c_ll, [_c_int, _c_int, _c_int]),
    "sx_attention_set_impl": (_c_int, [_c_int]),
    "sx_stream_copy": (_c_int, [_vp, _vp, _c_ll, _c_int, _vp, _vp, _vp]),
    "sx_kv_compact": (_c_int, [_vp, _vp, _c_int, _c_ll, _c_ll, _c_int, _vp, _vp, _c_int, _vp]),
    # fp32 target mode
    "sx_gemm_f32": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_ll, _c_int, _vp]),
    "sx_tree_attention_f32": (
        _c_int,
        [_vp, _vp, _vp, _c_ll, _vp, _c_int, _vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp],
    ),
    "sx_embed_f32": (_c_int, [_vp, _vp, _c_int, _c_int, _vp, _vp]),
    "sx_add_rmsnorm_f32": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, ctypes.c_float, _vp, _vp]),
    "sx_rope_kv_f32": (
        _c_int,
        [_vp, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _c_ll, _vp],
    ),
    "sx_kv_compact_f32": (_c_int, [_vp, _vp, _c_int, _c_ll, _c_ll, _c_int, _vp, _vp, _c_int, _vp]),
}

ROWS_LOGITS_F32, ROWS_PROBS_F64, ROWS_ARGMAX_PACKED = 0, 1, 2
SCORE_RAW, SCORE_ARGMAX, SCORE_WARP = 0, 1, 2

EPI_BF16, EPI_F32, EPI_ADD_F32, EPI_SWIGLU_BF16, EPI_SWIGLU_IL, EPI_RS_BF16, EPI_QKV_ROPE = 0, 1, 2, 3, 4, 5, 6

_lib = None


class SxError(RuntimeError):
    """A CUDA error reported by the native library."""


def load(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"native library {p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (load().sx_last_error() or b"").decode(errors="replace")
    if status < 0:
        raise ValueError(f"{what}: {msg}")
    raise SxError(f"{what}: CUDA error {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None stays None)."""
    if t is None:
        return None
    return int(t.data_ptr())
