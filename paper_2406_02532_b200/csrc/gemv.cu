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
// TMA-fed path (the default): one CTA per SM; a producer warp streams weight-row
// segments into a 9-stage shared-memory ring with 1-D bulk copies (no register
// cost per byte in flight: 144 KB per SM), the token rows stay resident in
// shared memory, 8 consumer warps form the dot products.
//   work item = (group, K chunk): group = 2 row pairs of one 128-row tile, rows
//   (2j, 2j+1, 2j+64, 2j+65), i.e. the RoPE / SwiGLU-IL pairs; chunk = 2048
//   columns. Groups are dealt round-robin to the CTAs (2-pair groups keep the
//   last round >= 0.96 full on every 7B / 70B shape).
//   consumer warp w: pair w >> 2, column quarter w & 3 of each chunk; at the end
//   of a group the 4 quarter sums are added in order (deterministic) and the
//   quarter-0 warp applies the epilogue.
// The producer issues the first ring of weight copies BEFORE griddepcontrol.wait
// (launched with programmatic stream serialization): the weights stream while
// the kernel that produces X finishes.
constexpr int kTmaConsumers = 8;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;
constexpr int kTmaKC = 2048;
constexpr int kTmaStages = 9;
constexpr int kTmaStageBytes = 4 * kTmaKC * 2;
constexpr int kTmaXMax = 64 * 1024;
constexpr int kTmaSmem = kTmaXMax + kTmaStages * kTmaStageBytes + 1024;

SX_DEV void tma_item(const GemvArgs& g, int i, int nchunk, int& tile, int& j, int& c0, int& kc) {
  const int grp = blockIdx.x + (i / nchunk) * gridDim.x;
  const int c = i % nchunk;
  tile = grp >> 5;
  j = grp & 31;
  c0 = c * kTmaKC;
  kc = min(kTmaKC, g.K - c0);
}

SX_DEV float dot_bf16x8(const uint4& w, const uint4& x, float acc) { return dot8(w, x, acc); }

template <int MT>
__global__ void __launch_bounds__(kTmaThreads, 1) gemv_tma_kernel(GemvArgs g) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* xs = smem_raw;                                   // [M][K] bf16 token rows
  uint8_t* ring = smem_raw + kTmaXMax;                       // [S][4][KC] bf16 weight segments
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kTmaStages * kTmaStageBytes);
  uint64_t* empty = full + kTmaStages;
  uint64_t* xbar = empty + kTmaStages;
  float* red = reinterpret_cast<float*>(xbar + 1);           // [8 warps][2 rows][MT]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (g.Nf + 127) / 128, groups = tiles * 32;
  const int nchunk = (g.K + kTmaKC - 1) / kTmaKC;
  const int my_groups = blockIdx.x < groups ? (groups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int n_items = my_groups * nchunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
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
      auto issue = [&](int i) {
        const int s = i % kTmaStages;
        if (i >= kTmaStages) mbar_wait(&empty[s], ((i / kTmaStages) & 1) ^ 1);
        int tile, j, c0, kc;
        tma_item(g, i, nchunk, tile, j, c0, kc);
        const int rows[4] = {tile * 128 + 2 * j, tile * 128 + 2 * j + 1, tile * 128 + 64 + 2 * j,
                             tile * 128 + 65 + 2 * j};
        uint32_t bytes = 0;
        for (int q = 0; q < 4; ++q) bytes += rows[q] < g.Nf ? (uint32_t)kc * 2 : 0u;
        mbar_arrive_expect_tx(&full[s], bytes);
        for (int q = 0; q < 4; ++q)
          if (rows[q] < g.Nf)
            bulk_load(ring + s * kTmaStageBytes + q * kTmaKC * 2, g.W + (long long)rows[q] * g.K + c0,
                      (uint32_t)kc * 2, &full[s], pol_w);
      };
      int i = 0;
      for (; i < n_items && i < kTmaStages; ++i) issue(i);  // weights do not depend on the previous kernel
      griddep_wait();
      mbar_arrive_expect_tx(xbar, (uint32_t)(g.M * g.K * 2));
      for (int t = 0; t < g.M; ++t)
        bulk_load(xs + (long long)t * g.K * 2, g.X + (long long)t * g.K, (uint32_t)g.K * 2, xbar, pol_x);
      for (; i < n_items; ++i) issue(i);
    }
    griddep_launch_dependents();
    return;
  }
  // ---------------- consumers ----------------
  griddep_wait();  // outputs (and the residual the ADD epilogue reads) are ordered after the previous kernel
  griddep_launch_dependents();
  const int pair = warp >> 2, q = warp & 3;
  mbar_wait(xbar, 0);
  float a0[MT], a1[MT];
#pragma unroll
  for (int t = 0; t < MT; ++t) a0[t] = a1[t] = 0.f;
  for (int i = 0; i < n_items; ++i) {
    const int s = i % kTmaStages;
    int tile, j, c0, kc;
    tma_item(g, i, nchunk, tile, j, c0, kc);
    mbar_wait(&full[s], (i / kTmaStages) & 1);
    const int qlen = kc >> 2, qv = qlen >> 3;  // columns / 16-byte vectors in this warp's quarter
    const uint4* w0 = reinterpret_cast<const uint4*>(ring + s * kTmaStageBytes + pair * kTmaKC * 2) + (q * qlen >> 3);
    const uint4* w1 = reinterpret_cast<const uint4*>(ring + s * kTmaStageBytes + (2 + pair) * kTmaKC * 2) + (q * qlen >> 3);
    const int f0 = tile * 128 + 2 * j + pair;
    const bool ok0 = f0 < g.Nf, ok1 = f0 + 64 < g.Nf;
    for (int v = lane; v < qv; v += 32) {
      const uint4 wa = ok0 ? w0[v] : make_uint4(0, 0, 0, 0);
      const uint4 wb = ok1 ? w1[v] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        if (t < g.M) {
          const uint4 xv = reinterpret_cast<const uint4*>(xs + (long long)t * g.K * 2)[(c0 + q * qlen) / 8 + v];
          a0[t] = dot_bf16x8(wa, xv, a0[t]);
          a1[t] = dot_bf16x8(wb, xv, a1[t]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (c0 + kc == g.K) {  // last chunk of the group: quarter sums -> epilogue
#pragma unroll
      for (int t = 0; t < MT; ++t) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a0[t] += __shfl_xor_sync(0xffffffffu, a0[t], o);
          a1[t] += __shfl_xor_sync(0xffffffffu, a1[t], o);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          red[(warp * 2 + 0) * MT + t] = a0[t];
          red[(warp * 2 + 1) * MT + t] = a1[t];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kTmaConsumers * 32) : "memory");
      if (q == 0 && lane < MT && lane < g.M) {
        float x0 = 0.f, x1 = 0.f;
        for (int qq = 0; qq < 4; ++qq) {  // fixed order
          x0 += red[((pair * 4 + qq) * 2 + 0) * MT + lane];
          x1 += red[((pair * 4 + qq) * 2 + 1) * MT + lane];
        }
        gemv_store(g, lane, tile, 2 * j + pair, x0, x1);
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kTmaConsumers * 32) : "memory");  // red is rewritten by the next group
#pragma unroll
      for (int t = 0; t < MT; ++t) a0[t] = a1[t] = 0.f;
    }
  }
}

static int g_gemv_enabled = 1;
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

template <int MT>
static int launch_gemv_tma_t(const GemvArgs& g, cudaStream_t stream) {
  if (int st = ensure_smem_attr((const void*)gemv_tma_kernel<MT>, kTmaSmem)) return st;
  const int groups = ((g.Nf + 127) / 128) * 32;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(groups < kNumSMs ? groups : kNumSMs));
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = kTmaSmem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_gemv_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemv_tma_kernel<MT>, g);
  SX_CHECK_LAUNCH("gemv_tma_kernel");
  return SX_OK;
}

int launch_gemv(const GemvArgs& g, cudaStream_t stream) {
  if ((reinterpret_cast<uintptr_t>(g.W) & 15) || (reinterpret_cast<uintptr_t>(g.X) & 15) || (g.K % 8))
    return arg_error("sx_gemm (thin): W / X must be 16-byte aligned and K a multiple of 8");
  if ((long long)g.M * g.K * 2 <= kTmaXMax && g.K % 64 == 0 && g_gemv_tma) {
    if (g.M == 1) return launch_gemv_tma_t<1>(g, stream);
    if (g.M == 2) return launch_gemv_tma_t<2>(g, stream);
    return launch_gemv_tma_t<4>(g, stream);
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
