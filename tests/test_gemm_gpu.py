"""KG tcgen05 GEMM vs a plain PyTorch fp32 reference of the same op."""

import pytest
import torch

from paper_2406_02532_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _ref(x, w):
    return x.float() @ w.float().t()


@pytest.mark.parametrize(
    "M,N,Kd",
    [(1, 128, 64), (17, 256, 128), (64, 4096, 4096), (100, 384, 512), (1025, 1024, 1024), (300, 1000, 192)],
)
def test_gemm_bf16_and_f32(cuda, M, N, Kd):
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    ref = _ref(x, w)
    y32 = K.gemm(x, w, epi=K.EPI_F32)
    torch.cuda.synchronize()
    tol = 1e-3 * (Kd ** 0.5)
    assert (y32 - ref).abs().max().item() < tol
    y16 = K.gemm(x, w, epi=K.EPI_BF16)
    assert (y16.float() - ref).abs().max().item() < tol + ref.abs().max().item() * 1e-2


@pytest.mark.parametrize("splits", [1, 2, 4])
def test_gemm_residual_add_and_splitk(cuda, splits):
    M, N, Kd = 48, 512, 2048
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.03).bfloat16()
    resid = torch.randn(M, N, generator=g, device=cuda)
    expect = resid + _ref(x, w)
    K.gemm(x, w, out=resid, epi=K.EPI_ADD_F32, splits=splits)
    torch.cuda.synchronize()
    assert (resid - expect).abs().max().item() < 5e-3


@pytest.mark.parametrize("M,splits", [(64, 0), (257, 1), (16, 4)])
def test_gemm_swiglu_dual(cuda, M, splits):
    N, Kd = 640, 1024
    g = torch.Generator(device=cuda).manual_seed(M)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    wg = (torch.randn(N, Kd, generator=g, device=cuda) * 0.03).bfloat16()
    wu = (torch.randn(N, Kd, generator=g, device=cuda) * 0.03).bfloat16()
    y = K.gemm(x, wg, epi=K.EPI_SWIGLU_BF16, w2=wu, splits=splits)
    gate = _ref(x, wg)
    up = _ref(x, wu)
    ref = torch.nn.functional.silu(gate) * up
    torch.cuda.synchronize()
    assert (y.float() - ref).abs().max().item() < 2e-2 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("M,N,Kd", [(256, 256, 64), (1025, 1280, 512), (300, 1000, 192), (64, 512, 256)])
def test_gemm_pair_vs_single(cuda, mode, M, N, Kd):
    from paper_2406_02532_b200 import _lib

    _lib.call("sx_gemm_set_pair_mode", mode)
    try:
        g = torch.Generator(device=cuda).manual_seed(M + N)
        x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
        w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
        w2 = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
        ref = _ref(x, w)
        y32 = K.gemm(x, w, epi=K.EPI_F32, splits=1)
        resid = torch.randn(M, N, generator=g, device=cuda)
        exp_r = resid + ref
        K.gemm(x, w, out=resid, epi=K.EPI_ADD_F32, splits=1)
        sw = K.gemm(x, w, epi=K.EPI_SWIGLU_BF16, w2=w2, splits=1)
        torch.cuda.synchronize()
        assert (y32 - ref).abs().max().item() < 1e-3 * Kd ** 0.5
        assert (resid - exp_r).abs().max().item() < 1e-3 * Kd ** 0.5
        ref_sw = torch.nn.functional.silu(ref) * _ref(x, w2)
        assert (sw.float() - ref_sw).abs().max().item() < 2e-2 * max(1.0, ref_sw.abs().max().item())
    finally:
        _lib.call("sx_gemm_set_pair_mode", 0)  # library default: auto


@pytest.mark.parametrize("sched", [1, 2, 3, 4, 0])
@pytest.mark.parametrize("M,N,Kd,dual", [(1025, 8192, 1024, False), (1025, 4480, 512, True), (200, 3072, 2048, False),
                                          (96, 1024, 4096, True)])
def test_gemm_schedules_agree(cuda, sched, M, N, Kd, dual):
    """whole tiles / stream-K / waves + split tail give the reference result;
    repeated launches (re-armed stream-K flags) are bit-identical."""
    g = torch.Generator(device=cuda).manual_seed(M * 3 + N)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.04).bfloat16()
    w2 = (torch.randn(N, Kd, generator=g, device=cuda) * 0.04).bfloat16() if dual else None
    epi = K.EPI_SWIGLU_BF16 if dual else K.EPI_F32
    a = K.gemm(x, w, epi=epi, w2=w2, splits=sched)
    b = K.gemm(x, w, epi=epi, w2=w2, splits=sched)
    ref = _ref(x, w)
    if dual:
        ref = torch.nn.functional.silu(ref) * _ref(x, w2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    tol = 2e-2 * max(1.0, ref.abs().max().item()) if dual else 1e-3 * Kd ** 0.5
    assert (a.float() - ref).abs().max().item() < tol


def test_gemm_large_perf_smoke(cuda):
    # 70B-shaped projection over a K=1024 tree (N = K+1 = 1025 tokens).
    M, N, Kd = 1025, 8192, 8192
    x = torch.randn(M, Kd, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, device=cuda) * 0.02).bfloat16()
    y = K.gemm(x, w, epi=K.EPI_BF16)
    torch.cuda.synchronize()
    ref = _ref(x, w)
    assert (y.float() - ref).abs().max().item() < 0.05
    for _ in range(3):
        K.gemm(x, w, out=y, epi=K.EPI_BF16)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        K.gemm(x, w, out=y, epi=K.EPI_BF16)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    tflops = 2 * M * N * Kd / ms / 1e9
    print(f"\n[gemm] 1025x8192x8192: {ms:.3f} ms  {tflops:.0f} TFLOP/s")


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("sched", [0, 1, 2, 3])
@pytest.mark.parametrize("M,F,Kd", [(1025, 2048, 512), (256, 1408, 1024), (40, 512, 256), (300, 704, 256)])
def test_gemm_swiglu_interleaved(cuda, mode, sched, M, F, Kd):
    """SX_EPI_SWIGLU_IL: one GEMM over [gate; up] interleaved in 64-row blocks
    (llama.interleave_gate_up) == silu(x gate^T) * (x up^T), every tile shape /
    schedule (stream-K partials are summed before the exchange)."""
    from paper_2406_02532_b200 import _lib
    from paper_2406_02532_b200.llama import interleave_gate_up

    _lib.call("sx_gemm_set_pair_mode", mode)
    try:
        g = torch.Generator(device=cuda).manual_seed(M * 7 + F)
        x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
        wg = (torch.randn(F, Kd, generator=g, device=cuda) * 0.05).bfloat16()
        wu = (torch.randn(F, Kd, generator=g, device=cuda) * 0.05).bfloat16()
        y = K.gemm(x, interleave_gate_up(wg, wu), epi=K.EPI_SWIGLU_IL, splits=sched)
        ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
        torch.cuda.synchronize()
        assert y.shape == (M, F)
        assert (y.float() - ref).abs().max().item() < 2e-2 * max(1.0, ref.abs().max().item())
        # same rounding as the dual-accumulator epilogue (identical fp32 sums in the plain schedule)
        if sched == 1:
            yd = K.gemm(x, wg, epi=K.EPI_SWIGLU_BF16, w2=wu, splits=1)
            assert (y.float() - yd.float()).abs().max().item() <= 1e-2 * max(1.0, ref.abs().max().item())
    finally:
        _lib.call("sx_gemm_set_pair_mode", 0)


@pytest.mark.parametrize("epi", [K.EPI_BF16, K.EPI_F32])
@pytest.mark.parametrize("M,N,Kd,ldo", [(1025, 1003, 256, 1024), (300, 4000, 512, 4000), (17, 520, 128, 1001)])
def test_gemm_strided_output_edges(cuda, epi, M, N, Kd, ldo):
    """Output into a wider row-strided buffer (vectorised 16-B epilogue when the
    rows are 16-B aligned, partial last feature group, scalar path otherwise);
    columns past N stay untouched."""
    g = torch.Generator(device=cuda).manual_seed(M + N + ldo)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    dt = torch.float32 if epi == K.EPI_F32 else torch.bfloat16
    buf = torch.full((M, ldo), 7.0, dtype=dt, device=cuda)
    K.gemm(x, w, out=buf[:, :N], epi=epi)
    torch.cuda.synchronize()
    ref = _ref(x, w)
    tol = 1e-3 * Kd ** 0.5 if epi == K.EPI_F32 else 2e-2 * max(1.0, ref.abs().max().item())
    assert (buf[:, :N].float() - ref).abs().max().item() < tol
    assert (buf[:, N:] == 7.0).all()


@pytest.mark.parametrize("mc", [0, 2, 4])
@pytest.mark.parametrize("M,N,Kd,epi", [(128, 4096, 1024, K.EPI_BF16), (256, 2944, 512, K.EPI_F32), (96, 1408, 256, K.EPI_SWIGLU_IL),
                                        (200, 1000, 384, K.EPI_BF16)])
def test_gemm_token_multicast_clusters(cuda, mc, M, N, Kd, epi):
    """Single-CTA tiles in clusters of mc CTAs sharing the token tile through TMA
    multicast (req bits 16-18; 0 = the planner's choice), incl. ragged clusters
    (N not a multiple of mc x 128 rows)."""
    from paper_2406_02532_b200.llama import split_gate_up

    g = torch.Generator(device=cuda).manual_seed(M * 3 + N + mc)
    x = torch.randn(M, Kd, generator=g, device=cuda).bfloat16()
    w = (torch.randn(N, Kd, generator=g, device=cuda) * 0.05).bfloat16()
    req = (1 | (1 << 4) | (mc << 16)) if mc else 0  # whole tiles, single-CTA, forced multicast width
    y = K.gemm(x, w, epi=epi, splits=req)
    torch.cuda.synchronize()
    if epi == K.EPI_SWIGLU_IL:
        wg, wu = split_gate_up(w)
        ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
    else:
        ref = _ref(x, w)
    tol = 1e-3 * Kd ** 0.5 if epi == K.EPI_F32 else 2e-2 * max(1.0, ref.abs().max().item())
    assert (y.float() - ref).abs().max().item() < tol
