"""The C-ABI library loads (no GPU needed) and exports exactly what
include/specexec_b200.h declares; argument errors surface as ValueError without
touching a device."""

import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2406_02532_b200 import _lib

HDR = pathlib.Path(__file__).resolve().parents[1] / "include" / "specexec_b200.h"


def header_symbols():
    text = HDR.read_text()
    return sorted(set(re.findall(r"SX_API\s+[\w\s\*]+?\b(sx_\w+)\s*\(", text)))


def test_header_declares_symbols():
    syms = header_symbols()
    assert "sx_gemm_bf16" in syms and "sx_tree_round" in syms and "sx_verify_walk" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True, check=True)
    exported = set(re.findall(r"\bT (sx_\w+)", out.stdout))
    for s in header_symbols():
        assert s in exported, s
        assert hasattr(lib, s)
    # nothing else leaks out of the C ABI
    assert exported == set(header_symbols())


def test_python_binding_covers_header():
    assert set(_lib.SIGNATURES) == set(header_symbols())


def test_version_and_errors_without_gpu():
    lib = _lib.load()
    assert lib.sx_abi_version() == 1
    bn, sp, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong()
    st = lib.sx_gemm_plan(10, 10, 100, 0, 0, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws))
    assert st < 0 and b"multiple of 64" in lib.sx_last_error()
    with pytest.raises(ValueError):
        _lib.check(st, "sx_gemm_plan")
    assert lib.sx_tree_workspace_bytes(1024, 64, 32000, 16) > 0
    assert lib.sx_tree_workspace_bytes(0, 64, 32000, 16) < 0


def test_gemm_plan_tiles():
    lib = _lib.load()
    bn, sp, ws = ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong()
    assert lib.sx_gemm_plan(1025, 8192, 8192, 0, 0, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert bn.value % 16 == 0 and bn.value * ((1025 + bn.value - 1) // bn.value) < 1025 + 5 * 16
    # CTA-pair tiles (256 weight rows) on 74 pairs: the token-tile width with the
    # lowest (rounds x width): 6 x 176 (192 tiles, 3 rounds) beats 5 x 208 -> whole tiles
    assert sp.value == 1 and bn.value == 176
    # the same for the long-K down projection (K = 28672): whole 176-wide tiles
    # measured 2-4 % faster than 208-wide tiles + a K-split tail
    assert lib.sx_gemm_plan(1025, 8192, 28672, 0, 0, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert bn.value == 176 and sp.value == 1
    # a forced split tail (sched 3) on 208-wide tiles still plans the 74-pair tail split
    assert lib.sx_gemm_plan(1025, 8192, 28672, 0, 3 | 2 << 4 | 13 << 8, ctypes.byref(bn), ctypes.byref(sp),
                            ctypes.byref(ws)) == 0
    assert bn.value == 208 and sp.value == 74 and ws.value == 1024 + 74 * 2 * bn.value * 128
    # 112 x 9 = 1008 SwiGLU pair tiles fill 14 waves at 97% -> whole tiles
    assert lib.sx_gemm_plan(1025, 28672, 8192, 1, 0, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert sp.value == 1 and ws.value == 0
    # one token tile (draft shapes): whole tiles unless stream-K is requested (sched 2)
    assert lib.sx_gemm_plan(64, 4096, 4096, 0, 0, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert sp.value == 1 and ws.value == 0
    assert lib.sx_gemm_plan(64, 4096, 4096, 0, 2, ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert sp.value == 148 and ws.value == 1024 + 148 * bn.value * 128
    # few weight tiles -> narrower token tiles so that enough SMs stream weights
    assert bn.value == 32


def test_attention_split_workspace_sizing():
    """Key-split workspace (host logic, no GPU): needed only when the tcgen05
    grid (ceil(N / (128 / G)) x KVH CTAs) is smaller than the 148 SMs; counters
    (a fixed 1 KB header for up to 148 CTAs, independent of N so one workspace
    serves every shape) then up to 8 splits x 128 rows x 132 floats per CTA."""
    lib = _lib.load()
    assert lib.sx_tree_attention_ws_bytes(1025, 64, 8) == 0  # 65 x 8 = 520 CTAs
    assert lib.sx_tree_attention_ws_bytes(1024, 32, 32) == 0  # 8 x 32 = 256 CTAs
    one = lib.sx_tree_attention_ws_bytes(1, 64, 8)  # 8 CTAs -> 8 splits
    assert one == 1024 + 8 * 8 * 128 * 132 * 4
    mid = lib.sx_tree_attention_ws_bytes(256, 32, 32)  # 64 CTAs -> ceil(296 / 64) = 5 splits
    assert mid == 1024 + 64 * 5 * 128 * 132 * 4
    assert lib.sx_tree_attention_ws_bytes(0, 64, 8) == 0
    assert lib.sx_tree_attention_ws_bytes(4, 64, 7) == 0  # H not a multiple of KVH: no split path
