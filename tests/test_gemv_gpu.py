"""KG-thin (csrc/gemv.cu): the 1..4-token weight-streaming path behind
sx_gemm_bf16 / sx_gemm_qkv_rope, vs a plain PyTorch fp32 reference of the same
op and vs the tcgen05 tile kernel (sx_gemm_set_gemv(0)) on the same inputs."""

import pytest
import torch

from paper_2406_02532_b200 import _lib
from paper_2406_02532_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _ref(x, w):
    return x.float() @ w.float().t()


def _tile_path(fn):
    _lib.call("sx_gemm_set_gemv", 0)
    try:
        return fn()
    finally:
        _lib.call("sx_gemm_set_gemv", 1)


@pytest.mark.parametrize("M", [1, 2, 3, 4])
@pytest.mark.parametrize("N,Kd", [(4096, 4096), (1003, 512), (32000, 256), (384, 11008)])
def test_gemv_bf16_f32_add(cuda, M, N, Kd):
    g = torch.Generator(device=cuda).manual_seed(M * 131 + N + Kd)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    ref = _ref(x, w)
    tol = 1e-3 * Kd ** 0.5
    y32 = K.gemm(x, w, epi=K.EPI_F32)
    y32_tile = _tile_path(lambda: K.gemm(x, w, epi=K.EPI_F32))
    torch.cuda.synchronize()
    assert (y32 - ref).abs().max().item() < tol
    assert (y32 - y32_tile).abs().max().item() < tol
    y16 = K.gemm(x, w, epi=K.EPI_BF16)
    assert (y16.float() - ref).abs().max().item() < tol + ref.abs().max().item() * 1e-2
    resid = torch.randn(M, N, generator=g, device=cuda)
    expect = resid + ref
    K.gemm(x, w, out=resid, epi=K.EPI_ADD_F32)
    torch.cuda.synchronize()
    assert (resid - expect).abs().max().item() < tol


@pytest.mark.parametrize("M", [1, 3])
def test_gemv_strided_output(cuda, M):
    N, Kd, ldo = 1000, 256, 1024
    g = torch.Generator(device=cuda).manual_seed(M)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    buf = torch.full((M, ldo), 7.0, device=cuda)
    K.gemm(x, w, out=buf[:, :N], epi=K.EPI_F32)
    torch.cuda.synchronize()
    assert (buf[:, :N] - _ref(x, w)).abs().max().item() < 1e-3 * Kd ** 0.5
    assert (buf[:, N:] == 7.0).all()


@pytest.mark.parametrize("M", [1, 2, 4])
@pytest.mark.parametrize("F,Kd", [(11008, 4096), (704, 256)])
def test_gemv_swiglu_interleaved(cuda, M, F, Kd):
    from paper_2406_02532_b200.llama import interleave_gate_up

    g = torch.Generator(device=cuda).manual_seed(M * 7 + F)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    wg = (torch.randn(F, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    wu = (torch.randn(F, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    wil = interleave_gate_up(wg, wu)
    y = K.gemm(x, wil, epi=K.EPI_SWIGLU_IL)
    yt = _tile_path(lambda: K.gemm(x, wil, epi=K.EPI_SWIGLU_IL))
    ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
    torch.cuda.synchronize()
    scale = max(1.0, ref.abs().max().item())
    assert y.shape == (M, F)
    assert (y.float() - ref).abs().max().item() < 2e-2 * scale
    assert (y.float() - yt.float()).abs().max().item() < 2e-2 * scale


@pytest.mark.parametrize("M", [1, 2, 4])
def test_gemv_qkv_rope_matches_tile_kernel(cuda, M):
    """RoPE (rotate-half) + K / V cache scatter from registers == the tile kernel's
    epilogue from the TMEM accumulators (bf16 rounding)."""
    H, KVH, Kd, slots, max_pos = 4, 2, 512, 64, 256
    g = torch.Generator(device=cuda).manual_seed(M + 11)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn((H + 2 * KVH) * 128, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    inv = 1.0 / (10000.0 ** (torch.arange(0, 64, device=cuda, dtype=torch.float32) / 64))
    ang = torch.arange(max_pos, device=cuda, dtype=torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos().contiguous(), ang.sin().contiguous()
    pos = torch.tensor([37, 5, 100, 3][:M], dtype=torch.int32, device=cuda)
    slot = torch.tensor([9, 40, 2, 63][:M], dtype=torch.int32, device=cuda)

    def run():
        q = torch.zeros(M, H, 128, dtype=torch.bfloat16, device=cuda)
        kc = torch.zeros(KVH, slots, 128, dtype=torch.bfloat16, device=cuda)
        vc = torch.zeros_like(kc)
        K.gemm_qkv_rope(x, w, H, KVH, pos, 0, slot, 0, cos, sin, q, kc, vc, slots)
        return q, kc, vc

    a = run()
    b = _tile_path(run)
    torch.cuda.synchronize()
    for u, v in zip(a, b):
        assert (u.float() - v.float()).abs().max().item() <= 2e-2 * max(1.0, v.float().abs().max().item())
    # untouched slots stay zero
    mask = torch.ones(slots, dtype=torch.bool, device=cuda)
    mask[slot.long()] = False
    assert (a[1][:, mask] == 0).all() and (a[2][:, mask] == 0).all()


@pytest.mark.parametrize("M,N,Kd", [(1, 1024, 28672), (2, 512, 28672), (4, 1003, 8192), (1, 130, 64)])
def test_gemv_long_k_and_fallback(cuda, M, N, Kd):
    """Token rows resident in shared memory up to 64 KB (70B down projection at
    M = 1: 57 KB), the register-load fallback beyond it (M = 2, K = 28672),
    partial 128-row tiles and a single K chunk shorter than the stage."""
    g = torch.Generator(device=cuda).manual_seed(M + N + Kd)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.02).bfloat16()
    ref = _ref(x, w)
    y = K.gemm(x, w, epi=K.EPI_F32)
    yt = _tile_path(lambda: K.gemm(x, w, epi=K.EPI_F32))
    torch.cuda.synchronize()
    tol = 1e-3 * Kd ** 0.5
    assert (y - ref).abs().max().item() < tol
    assert (y - yt).abs().max().item() < tol


def test_gemv_deterministic(cuda):
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.randn(1, 4096, generator=g, device=cuda).bfloat16()
    w = (torch.randn(12288, 4096, generator=g, device=cuda) * 0.02).bfloat16()
    a = K.gemm(x, w, epi=K.EPI_F32)
    b = K.gemm(x, w, epi=K.EPI_F32)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
