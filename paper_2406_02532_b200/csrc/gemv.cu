// KG-thin: weight-streaming projection for 1..4 tokens (the draft's root round,
// one-token chain / sequential-decoding steps). At M <= 4 the projection is a
// matrix-vector product bound by the weight bytes (2 N K), not by the tensor
// pipe: the tcgen05 tile kernel pads the tokens to 16, and its per-tile
// prologue / TMA ring / TMEM epilogue round trips cap a single launch at
// 1.6-3.9 TB/s on the 7B draft shapes (tools/draft_probe.py); a register-load
// warp-per-row kernel reached only 2.3-4.7 TB/s (ncu, profiles/r2) -- the
// bytes in flight per SM are bounded by registers / L1 miss slots.
// The default path (gemv_tma_kernel) streams the weights with 1-D bulk copies
// (cp.async.bulk, mbarrier ring) into shared memory, 144 KB in flight per SM,
// with the token rows resident in shared memory; the register-load kernel is
// the fallback when the token rows do not fit (M x K x 2 > 64 KB).
// Both work on weight-row PAIRS (f, f + 64) of a 128-row tile -- the pairs the
// RoPE (rotate-half) and interleaved-SwiGLU epilogues combine -- so every
// epilogue of the tile kernel (bf16, fp32, fp32 residual add, SwiGLU-IL,
// QKV + RoPE + KV scatter; gemm_tc.cu epilogue_store) is applied from
// registers. fp32 accumulation; the summation order differs from the tile
// kernel's (fp32 rounding only) and is fixed (deterministic).
#include <cstdlib>

#include "capi_util.h"
#include "common.cuh"
#include "gemv.h"
#include "specexec_b200.h"

namespace sx {

constexpr int kGemvThreads = 256;
constexpr int kGemvUnroll = 8;

SX_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

SX_DEV float dot8(const uint4& w, const uint4& x, float acc) {
  const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&w);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 fa = __bfloat1622float2(a[i]), fb = __bfloat1622float2(b[i]);
    acc = fmaf(fa.x, fb.x, acc);
    acc = fmaf(fa.y, fb.y, acc);
  }
  return acc;
}

SX_DEV float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Epilogue of one weight-row pair (rows tile*128 + r and + 64) for token t.
SX_DEV void gemv_store(const GemvArgs& g, int t, int tile, int r, float x0, float x1) {
  const int f0 = tile * 128 + r, f1 = f0 + 64;
  const bool ok0 = f0 < g.Nf, ok1 = f1 < g.Nf;
  switch (g.epi) {
    case SX_EPI_BF16: {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out) + (long long)t * g.ldo;
      if (ok0) o[f0] = __float2bfloat16(x0);
      if (ok1) o[f1] = __float2bfloat16(x1);
      break;
    }
    case SX_EPI_F32: {
      float* o = reinterpret_cast<float*>(g.out) + (long long)t * g.ldo;
      if (ok0) o[f0] = x0;
      if (ok1) o[f1] = x1;
      break;
    }
    case SX_EPI_ADD_F32: {
      float* o = reinterpret_cast<float*>(g.out) + (long long)t * g.ldo;
      if (ok0) o[f0] += x0;
      if (ok1) o[f1] += x1;
      break;
    }
    case SX_EPI_SWIGLU_IL: {  // rows r (gate) and r + 64 (up) of the tile -> output feature tile*64 + r
      if (ok1) {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out) + (long long)t * g.ldo;
        o[tile * 64 + r] = __float2bfloat16(silu_f(x0) * x1);
      }
      break;
    }
    default: {  // SX_EPI_QKV_ROPE: tile = head, rows (d, d + 64) = the rotate-half pair
      const int hh = tile;
      const long long sl = g.rope_slot_base + (g.rope_slot ? g.rope_slot[t] : t);
      __nv_bfloat16* dst;
      if (hh < g.rope_H)
        dst = g.rope_q + ((long long)t * g.rope_H + hh) * 128;
      else if (hh < g.rope_H + g.rope_KVH)
        dst = g.rope_kc + ((long long)(hh - g.rope_H) * g.rope_slots + sl) * 128;
      else
        dst = g.rope_vc + ((long long)(hh - g.rope_H - g.rope_KVH) * g.rope_slots + sl) * 128;
      float lo = x0, hi = x1;
      if (hh < g.rope_H + g.rope_KVH) {
        const long long pos = g.rope_pos_base + (g.rope_pos ? g.rope_pos[t] : t);
        const float c = g.rope_cos[pos * 64 + r], s = g.rope_sin[pos * 64 + r];
        lo = x0 * c - x1 * s;
        hi = x1 * c + x0 * s;
      }
      dst[r] = __float2bfloat16(lo);
      dst[r + 64] = __float2bfloat16(hi);
      break;
    }
  }
}

// Fallback (token rows too large to keep in shared memory): one warp per row pair,
// 16-byte register loads.
template <int MT>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvArgs g) {
  const int lane = threadIdx.x & 31;
  const int warp0 = blockIdx.x * (kGemvThreads / 32) + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * (kGemvThreads / 32);
  const int pairs = ((g.Nf + 127) / 128) * 64;
  const int K8 = g.K / 8;  // 16-byte vectors per weight row
  const uint4 zero = make_uint4(0, 0, 0, 0);
  // Launched with programmatic stream serialization: the weights do not depend
  // on the preceding kernel, so each warp pulls its first row pair into L2 while
  // the producer of X (norm / attention / the previous projection) finishes.
  if (lane == 0 && warp0 < pairs) {
    const int f = (warp0 >> 6) * 128 + (warp0 & 63);
    if (f < g.Nf) bulk_prefetch_l2(g.W + (long long)f * g.K, (uint32_t)g.K * 2);
    if (f + 64 < g.Nf) bulk_prefetch_l2(g.W + (long long)(f + 64) * g.K, (uint32_t)g.K * 2);
  }
  griddep_wait();
  griddep_launch_dependents();
  for (int p = warp0; p < pairs; p += nwarps) {
    const int tile = p >> 6, r = p & 63;
    const int f0 = tile * 128 + r, f1 = f0 + 64;
    const bool ok0 = f0 < g.Nf, ok1 = f1 < g.Nf;
    const uint4* w0 = reinterpret_cast<const uint4*>(g.W) + (long long)f0 * K8;
    const uint4* w1 = reinterpret_cast<const uint4*>(g.W) + (long long)f1 * K8;
    float a0[MT], a1[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) a0[t] = a1[t] = 0.f;
    for (int kb = lane; kb < K8; kb += 32 * kGemvUnroll) {
      uint4 wa[kGemvUnroll], wb[kGemvUnroll];
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        const int k = kb + u * 32;
        wa[u] = (ok0 && k < K8) ? ld_stream16(w0 + k) : zero;
        wb[u] = (ok1 && k < K8) ? ld_stream16(w1 + k) : zero;
      }
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        const int k = kb + u * 32;
        if (k < K8) {
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            if (t < g.M) {
              const uint4 xv = __ldg(reinterpret_cast<const uint4*>(g.X) + (long long)t * K8 + k);
              a0[t] = dot8(wa[u], xv, a0[t]);
              a1[t] = dot8(wb[u], xv, a1[t]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0[t] += __shfl_xor_sync(0xffffffffu, a0[t], o);
        a1[t] += __shfl_xor_sync(0xffffffffu, a1[t], o);
      }
    }
    if (lane < MT && lane < g.M) {  // lane t stores token t
      float x0 = 0.f, x1 = 0.f;
#pragma unroll
      for (int t = 0; t < MT; ++t)
        if (t == lane) x0 = a0[t], x1 = a1[t];
      gemv_store(g, lane, tile, r, x0, x1);
    }
  }
}


// ---------------------------------------------------------------------------
// TMA-fed path (the default): a producer warp streams weight-row segments into a
// shared-memory ring with 1-D bulk copies (no register cost per byte in flight),
// the token rows stay resident in shared memory, 8 consumer warps form the dot
// products.
//   Unit of work = a GROUP of 2 row pairs (f, f + 64) of one 128-row tile (the
//   RoPE / SwiGLU-IL pairs): rows 2j, 2j+1, 2j+64, 2j+65. Each CTA owns a
//   contiguous range of groups (groups / grid, +-1). A ring stage holds the 4
//   rows of a group over kGemvKC = 4096 columns: every bulk copy is one 8 KB
//   contiguous run of a weight row. Measured on B200 (tools/micro/stream_probe.cu,
//   profiles/r2/stream_probe.txt): row segments of 1 / 2 / 4 / 8 KB stream at
//   ~1.4 / 3.4 / 5.1 / 6.5 TB/s -- the segment length, not the bytes in flight,
//   sets the rate -- so the stage is whole 8 KB row runs, not narrow column chunks.
//   Consumer warp w: pair w >> 2, column quarter w & 3 of each stage; at the end
//   of a group the 4 quarter sums of a pair meet in shared memory (named barrier
//   of the pair's 4 warps, fixed order) and lane t of the quarter-0 warp stores
//   token t.
// The producer issues the first ring of weight copies BEFORE griddepcontrol.wait:
// the weights do not depend on the kernel that produces X.
constexpr int kTmaConsumers = 8;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;
constexpr int kGemvKC = 4096;
constexpr int kGemvStageBytes = 4 * kGemvKC * 2;

template <int S>
static int gemv_tma_smem(int M, int K) { return S * kGemvStageBytes + 1024 + ((M * K * 2 + 127) / 128) * 128; }

template <int MT, int S>
__global__ void __launch_bounds__(kTmaThreads, 1) gemv_tma_kernel(GemvArgs g) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = smem_raw;                                            // [S][4 rows][kGemvKC] bf16
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * kGemvStageBytes);
  uint64_t* empty = full + S;
  uint64_t* xbar = empty + S;
  float* red = reinterpret_cast<float*>(ring + S * kGemvStageBytes + 256);  // [2 parity][8 warps][2 rows][MT]
  uint8_t* xs = ring + S * kGemvStageBytes + 1024;                       // [M][K] bf16 token rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = ((g.Nf + 127) / 128) * 32;
  const int g_begin = (int)((long long)groups * blockIdx.x / gridDim.x);
  const int g_end = (int)((long long)groups * (blockIdx.x + 1) / gridDim.x);
  const int nchunk = (g.K + kGemvKC - 1) / kGemvKC;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers);
    }
    mbar_init(xbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == kTmaConsumers) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      auto load_x = [&]() {
        griddep_wait();
        mbar_arrive_expect_tx(xbar, (uint32_t)(g.M * g.K * 2));
        for (int t = 0; t < g.M; ++t)
          bulk_load(xs + (long long)t * g.K * 2, g.X + (long long)t * g.K, (uint32_t)g.K * 2, xbar, pol_x);
      };
      int s = 0, ph = 0, issued = 0;
      bool x_loaded = false;
      for (int gi = g_begin; gi < g_end; ++gi) {
        const int tile = gi >> 5, j = gi & 31;
        const int rows[4] = {tile * 128 + 2 * j, tile * 128 + 2 * j + 1, tile * 128 + 64 + 2 * j,
                             tile * 128 + 65 + 2 * j};
        for (int c0 = 0; c0 < g.K; c0 += kGemvKC) {
          if (issued == S) load_x(), x_loaded = true;  // the first ring is in flight: now wait for X's producer
          if (issued >= S) mbar_wait(&empty[s], ph ^ 1);
          const uint32_t seg = (uint32_t)min(kGemvKC, g.K - c0) * 2;
          uint32_t bytes = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) bytes += rows[q] < g.Nf ? seg : 0u;
          mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (rows[q] < g.Nf)
              bulk_load(ring + s * kGemvStageBytes + q * kGemvKC * 2, g.W + (long long)rows[q] * g.K + c0, seg,
                        &full[s], pol_w);
          ++issued;
          if (++s == S) s = 0, ph ^= 1;
        }
      }
      if (!x_loaded) load_x();  // the whole range fit in the first ring
    }
    griddep_launch_dependents();
    return;
  }
  // ---------------- consumers ----------------
  griddep_wait();  // outputs (and the residual the ADD epilogue reads) are ordered after the previous kernel
  griddep_launch_dependents();
  mbar_wait(xbar, 0);
  const int pair = warp >> 2, q = warp & 3;
  const int K8 = g.K >> 3;
  const uint4* xv0 = reinterpret_cast<const uint4*>(xs);
  int s = 0, ph = 0, par = 0;
  for (int gi = g_begin; gi < g_end; ++gi, par ^= 1) {
    float a0[MT], a1[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) a0[t] = a1[t] = 0.f;
    for (int c0 = 0; c0 < g.K; c0 += kGemvKC) {
      const int kc = min(kGemvKC, g.K - c0);
      const int qv = kc >> 5;  // 16-byte vectors in this warp's quarter (kc % 32 == 0)
      mbar_wait(&full[s], ph);
      const uint4* w0 = reinterpret_cast<const uint4*>(ring + s * kGemvStageBytes + pair * kGemvKC * 2) + q * qv;
      const uint4* w1 = reinterpret_cast<const uint4*>(ring + s * kGemvStageBytes + (2 + pair) * kGemvKC * 2) + q * qv;
      const uint4* xc = xv0 + ((c0 >> 3) + q * qv);
#pragma unroll 4
      for (int v = lane; v < qv; v += 32) {
        const uint4 wa = w0[v], wb = w1[v];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          if (t < g.M) {
            const uint4 x = xc[(long long)t * K8 + v];
            a0[t] = dot8(wa, x, a0[t]);
            a1[t] = dot8(wb, x, a1[t]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) s = 0, ph ^= 1;
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0[t] += __shfl_xor_sync(0xffffffffu, a0[t], o);
        a1[t] += __shfl_xor_sync(0xffffffffu, a1[t], o);
      }
    }
    float* rp = red + par * (kTmaConsumers * 2 * MT);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        rp[(warp * 2 + 0) * MT + t] = a0[t];
        rp[(warp * 2 + 1) * MT + t] = a1[t];
      }
    }
    // the 4 warps of this pair; red is double-buffered by group parity, so no second barrier
    asm volatile("bar.sync %0, 128;" ::"r"(1 + pair) : "memory");
    if (q == 0 && lane < MT && lane < g.M) {
      float x0 = 0.f, x1 = 0.f;
      for (int qq = 0; qq < 4; ++qq) {  // fixed order
        x0 += rp[((pair * 4 + qq) * 2 + 0) * MT + lane];
        x1 += rp[((pair * 4 + qq) * 2 + 1) * MT + lane];
      }
      const int tile = gi >> 5, j = gi & 31;
      gemv_store(g, lane, tile, 2 * j + pair, x0, x1);
    }
  }
}

// SX_GEMV=0: the tile kernel for every M (A/B); sx_gemm_set_gemv sets it at run time
static int g_gemv_enabled = getenv("SX_GEMV") ? atoi(getenv("SX_GEMV")) : 1;
// programmatic dependent launch (weights prefetched into L2 during the producer's tail); SX_GEMV_PDL=0 disables
static const int g_gemv_pdl = getenv("SX_GEMV_PDL") ? atoi(getenv("SX_GEMV_PDL")) : 1;
// SX_GEMV_TMA=0: the register-load fallback for every shape (A/B)
static const int g_gemv_tma = getenv("SX_GEMV_TMA") ? atoi(getenv("SX_GEMV_TMA")) : 1;

bool gemv_applies(int M, int epi, int dual) {
  if (!g_gemv_enabled || dual || M < 1 || M > kGemvMaxTokens) return false;
  return epi == SX_EPI_BF16 || epi == SX_EPI_F32 || epi == SX_EPI_ADD_F32 || epi == SX_EPI_SWIGLU_IL ||
         epi == SX_EPI_QKV_ROPE;
}

template <int MT>
static int launch_gemv_t(const GemvArgs& g, cudaStream_t stream) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_kernel<MT>, kGemvThreads, 0);
    if (occ < 1) occ = 1;
  }
  const long long pairs = (long long)((g.Nf + 127) / 128) * 64;
  const long long need = (pairs + kGemvThreads / 32 - 1) / (kGemvThreads / 32);
  const long long cap = (long long)occ * kNumSMs;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(need < cap ? need : cap));
  cfg.blockDim = dim3(kGemvThreads);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // griddepcontrol.wait in the kernel
  at[0].val.programmaticStreamSerializationAllowed = g_gemv_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemv_kernel<MT>, g);
  SX_CHECK_LAUNCH("gemv_kernel");
  return SX_OK;
}

// ring depth: SX_GEMV_STAGES = 4 (default, 128 KB) | 2 (64 KB: two CTAs per SM, the next projection co-resident)
static const int g_gemv_stages = getenv("SX_GEMV_STAGES") ? atoi(getenv("SX_GEMV_STAGES")) : 4;

template <int MT, int S>
static int launch_gemv_tma_t(const GemvArgs& g, cudaStream_t stream) {
  const int smem = gemv_tma_smem<S>(g.M, g.K);
  if (int st = ensure_smem_attr((const void*)gemv_tma_kernel<MT, S>, 227 * 1024)) return st;
  const int groups = ((g.Nf + 127) / 128) * 32;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(groups < kNumSMs ? groups : kNumSMs));
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_gemv_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemv_tma_kernel<MT, S>, g);
  SX_CHECK_LAUNCH("gemv_tma_kernel");
  return SX_OK;
}

template <int MT>
static int launch_gemv_tma_m(const GemvArgs& g, cudaStream_t stream) {
  if (g_gemv_stages == 2) return launch_gemv_tma_t<MT, 2>(g, stream);
  return launch_gemv_tma_t<MT, 4>(g, stream);
}

int launch_gemv(const GemvArgs& g, cudaStream_t stream) {
  if ((reinterpret_cast<uintptr_t>(g.W) & 15) || (reinterpret_cast<uintptr_t>(g.X) & 15) || (g.K % 8))
    return arg_error("sx_gemm (thin): W / X must be 16-byte aligned and K a multiple of 8");
  if ((long long)g.M * g.K * 2 <= 64 * 1024 && g.K % 32 == 0 && g_gemv_tma) {
    if (g.M == 1) return launch_gemv_tma_m<1>(g, stream);
    if (g.M == 2) return launch_gemv_tma_m<2>(g, stream);
    return launch_gemv_tma_m<4>(g, stream);
  }
  if (g.M == 1) return launch_gemv_t<1>(g, stream);
  if (g.M == 2) return launch_gemv_t<2>(g, stream);
  return launch_gemv_t<4>(g, stream);
}

}  // namespace sx

extern "C" int sx_gemm_set_gemv(int enabled) {
  if (enabled < 0 || enabled > 1) return sx::arg_error("sx_gemm_set_gemv: 0 (tile kernel only) or 1 (auto)");
  sx::g_gemv_enabled = enabled;
  return sx::SX_OK;
}
