// KG: bf16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   Y[t, f] = sum_k X[t, k] * W[f, k]        (X: tokens x K, W: features x K)
//
// The weight matrix is the MMA "A" operand (M = 128 features per tile) and the
// tokens are the "B" operand (N = BN tokens, any multiple of 16 up to 256), so
// the token count of a SpecExec pass (K+1 tree tokens, or a draft batch of B
// frontier nodes) is padded only to 16, not to 128. That is the shape of every
// projection of the target forward over the tree (stage 2) and of the draft
// forward per tree round (stage 1) -- the dense contractions behind the
// reference's `LanguageModel.next_distributions` (pkg/src/speckit/models.py:47-52).
//
// Structure: persistent, warp-specialised, one CTA per SM.
//   warp 0      TMA producer   (weights + tokens tiles, 128B swizzle, mbarrier ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue       (tcgen05.ld -> registers -> fused epilogue -> global)
// Accumulators are double-buffered in TMEM when they fit so the epilogue of one
// tile overlaps the main loop of the next.
//
// Epilogues: bf16 store, fp32 store (logits), fp32 residual add, and a fused
// SwiGLU "dual" mode where a second weight matrix (up-projection) is multiplied
// into a second accumulator and the epilogue writes silu(gate) * up.
// Split-K (for small-token, weight-streaming shapes that would otherwise leave
// SMs idle) writes fp32 partials that `splitk_reduce` sums in a fixed order
// (deterministic) before applying the same epilogue.
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"

namespace sx {

struct GemmArgs {
  int M, Nf, K;
  int BN;
  int tiles_f, tiles_t, splits, kb_per_split, kb_total, units;
  int epi, dual, stages;
  uint32_t stage_bytes, a_bytes, b_bytes;
  uint32_t acc_cols;  // TMEM columns per accumulator buffer
  int acc_stages;
  uint32_t tmem_cols;
  void* out;
  long long ldo;
  float* ws;
};

constexpr int kGemmThreads = 192;

SX_DEV float silu(float x) { return x / (1.0f + __expf(-x)); }

// TMEM accumulator (this thread's lane = feature f, BN token columns) -> global.
SX_DEV void epilogue_tile(const GemmArgs& g, uint32_t tbase, int f, bool fok, int tt, int split) {
  for (int c = 0; c < g.BN; c += 16) {
    uint32_t r[16];
    uint32_t r2[16];
    tmem_ld16(tbase + c, r);
    if (g.dual) tmem_ld16(tbase + g.BN + c, r2);
    tmem_ld_wait();
    const int t0 = tt * g.BN + c;
    if (g.splits > 1) {
      float* ws = g.ws + ((long long)split * (g.dual ? 2 : 1) * g.M) * g.Nf;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = t0 + j;
        if (t < g.M && fok) {
          ws[(long long)t * g.Nf + f] = __uint_as_float(r[j]);
          if (g.dual) ws[((long long)g.M + t) * g.Nf + f] = __uint_as_float(r2[j]);
        }
      }
    } else if (g.epi == SX_EPI_BF16) {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = t0 + j;
        if (t < g.M && fok) o[(long long)t * g.ldo + f] = __float2bfloat16(__uint_as_float(r[j]));
      }
    } else if (g.epi == SX_EPI_F32) {
      float* o = reinterpret_cast<float*>(g.out);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = t0 + j;
        if (t < g.M && fok) o[(long long)t * g.ldo + f] = __uint_as_float(r[j]);
      }
    } else if (g.epi == SX_EPI_ADD_F32) {
      float* o = reinterpret_cast<float*>(g.out);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = t0 + j;
        if (t < g.M && fok) o[(long long)t * g.ldo + f] += __uint_as_float(r[j]);
      }
    } else {  // SX_EPI_SWIGLU_BF16
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = t0 + j;
        if (t < g.M && fok) {
          const float gv = __uint_as_float(r[j]);
          o[(long long)t * g.ldo + f] = __float2bfloat16(silu(gv) * __uint_as_float(r2[j]));
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB, const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + g.stages * g.stage_bytes);
  uint64_t* empty_bar = full_bar + g.stages;
  uint64_t* tfull_bar = empty_bar + g.stages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id();
  const int lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    if (g.dual) tma_prefetch_desc(&mapA2);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, g.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t pol_w = policy_evict_first();  // weights stream through once per token tile group
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
        const int split = u % g.splits;
        const int rest = u / g.splits;
        const int tt = rest % g.tiles_t;
        const int tf = rest / g.tiles_t;
        const int kb0 = split * g.kb_per_split;
        const int kb1 = min(g.kb_total, kb0 + g.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * g.stage_bytes;
          mbar_arrive_expect_tx(&full_bar[stage], g.stage_bytes);
          tma_load_2d_hint(sa, &mapA, &full_bar[stage], kb * 64, tf * 128, pol_w);
          if (g.dual) tma_load_2d_hint(sa + g.a_bytes, &mapA2, &full_bar[stage], kb * 64, tf * 128, pol_w);
          tma_load_2d(sa + (g.dual ? 2 : 1) * g.a_bytes, &mapB, &full_bar[stage], kb * 64, tt * g.BN);
          if (++stage == g.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = idesc_bf16_f32(128, g.BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
        const int split = u % g.splits;
        const int kb0 = split * g.kb_per_split;
        const int kb1 = min(g.kb_total, kb0 + g.kb_per_split);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * g.acc_cols;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* sa = smem + stage * g.stage_bytes;
          const uint64_t da = smem_desc_k_sw128(sa);
          const uint64_t da2 = smem_desc_k_sw128(sa + g.a_bytes);
          const uint64_t db = smem_desc_k_sw128(sa + (g.dual ? 2 : 1) * g.a_bytes);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // advance 16 bf16 = 32 B along K inside the swizzle atom (>>4 => +2)
            const uint32_t acc_flag = (kb > kb0 || k > 0) ? 1u : 0u;
            tc_mma_bf16(d0, da + 2 * k, db + 2 * k, idesc, acc_flag);
            if (g.dual) tc_mma_bf16(d0 + g.BN, da2 + 2 * k, db + 2 * k, idesc, acc_flag);
          }
          tc_commit(&empty_bar[stage]);
          if (++stage == g.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull_bar[acc]);
        if (++acc == g.acc_stages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int split = u % g.splits;
      const int rest = u / g.splits;
      const int tt = rest % g.tiles_t;
      const int tf = rest / g.tiles_t;
      const int f = tf * 128 + quarter * 32 + lane;
      const bool fok = f < g.Nf;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * g.acc_cols;
      epilogue_tile(g, tbase, f, fok, tt, split);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == g.acc_stages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, g.tmem_cols);
  }
}

// ----------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2, M = 256 features per pair): each CTA
// stages its 128 weight rows and half of the BN token rows; the leader issues
// the pair MMA, so every token tile fetched from L2 feeds 256 features instead
// of 128 (operand traffic per FLOP drops ~1.5x: the single-CTA kernel is
// L2-bandwidth bound at M = 128). Used for the compute-bound target pass.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                    const __grid_constant__ CUtensorMap mapB, const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + g.stages * g.stage_bytes);
  uint64_t* empty_bar = full_bar + g.stages;
  uint64_t* tfull_bar = empty_bar + g.stages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int half = g.BN / 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    if (g.dual) tma_prefetch_desc(&mapA2);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_base_smem, g.tmem_cols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < g.units; u += npairs) {
        const int rest = u / g.splits;
        const int tt = rest % g.tiles_t;
        const int tf = rest / g.tiles_t;
        for (int kb = 0; kb < g.kb_total; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * g.stage_bytes;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * g.stage_bytes);
          const int frow = tf * 256 + (int)rank * 128;
          tma_load_2d_2sm(sa, &mapA, &full_bar[stage], kb * 64, frow, pol_w);
          if (g.dual) tma_load_2d_2sm(sa + g.a_bytes, &mapA2, &full_bar[stage], kb * 64, frow, pol_w);
          tma_load_2d_2sm(sa + (g.dual ? 2 : 1) * g.a_bytes, &mapB, &full_bar[stage], kb * 64,
                          tt * g.BN + (int)rank * half, pol_x);
          if (++stage == g.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, g.BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < g.units; u += npairs) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * g.acc_cols;
        for (int kb = 0; kb < g.kb_total; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* sa = smem + stage * g.stage_bytes;
          const uint64_t da = smem_desc_k_sw128(sa);
          const uint64_t da2 = smem_desc_k_sw128(sa + g.a_bytes);
          const uint64_t db = smem_desc_k_sw128(sa + (g.dual ? 2 : 1) * g.a_bytes);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc_flag = (kb > 0 || k > 0) ? 1u : 0u;
            tc_mma_bf16_2sm(d0, da + 2 * k, db + 2 * k, idesc, acc_flag);
            if (g.dual) tc_mma_bf16_2sm(d0 + g.BN, da2 + 2 * k, db + 2 * k, idesc, acc_flag);
          }
          tc_commit_2sm_mc(&empty_bar[stage], 0x3);
          if (++stage == g.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_2sm_mc(&tfull_bar[acc], 0x3);
        if (++acc == g.acc_stages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < g.units; u += npairs) {
      const int rest = u / g.splits;
      const int tt = rest % g.tiles_t;
      const int tf = rest / g.tiles_t;
      const int f = tf * 256 + (int)rank * 128 + quarter * 32 + lane;
      const bool fok = f < g.Nf;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * g.acc_cols;
      epilogue_tile(g, tbase, f, fok, tt, 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 0);
      if (++acc == g.acc_stages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, g.tmem_cols);
  }
}

// Deterministic split-K reduction: partial planes are summed in split order,
// then the epilogue of the GEMM is applied.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, void* out, long long ldo, int M, int Nf,
                                     int splits, int epi, int dual) {
  const long long total = (long long)M * Nf;
  const long long plane = (long long)(dual ? 2 : 1) * total;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i / Nf);
    const int f = (int)(i % Nf);
    float s = 0.f, s2 = 0.f;
    for (int k = 0; k < splits; ++k) {
      s += ws[k * plane + i];
      if (dual) s2 += ws[k * plane + total + i];
    }
    const long long o = (long long)t * ldo + f;
    if (epi == SX_EPI_BF16) {
      reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16(s);
    } else if (epi == SX_EPI_F32) {
      reinterpret_cast<float*>(out)[o] = s;
    } else if (epi == SX_EPI_ADD_F32) {
      reinterpret_cast<float*>(out)[o] += s;
    } else {
      reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16(silu(s) * s2);
    }
  }
}

// 0 = auto (pair for M >= 256), 1 = single-CTA only, 2 = pair whenever legal
static int g_pair_mode = 0;

// tuning overrides (read once): SX_GEMM_BN_CAP (token-tile cap), SX_GEMM_STAGES (max pipeline depth)
static int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}
static int bn_cap_single() {
  static int v = env_int("SX_GEMM_BN_CAP", 256);
  return v;
}
static int max_stages() {
  static int v = env_int("SX_GEMM_STAGES", 8);
  return v;
}

static int pick_bn(int M, int cap) {
  int tiles = (M + cap - 1) / cap;
  int bn = (M + tiles - 1) / tiles;
  bn = (bn + 15) / 16 * 16;
  if (bn < 16) bn = 16;
  return bn;
}

}  // namespace sx

using namespace sx;

extern "C" int sx_gemm_set_pair_mode(int mode) {
  if (mode < 0 || mode > 2) return arg_error("sx_gemm_set_pair_mode: mode must be 0, 1 or 2");
  g_pair_mode = mode;
  return SX_OK;
}

extern "C" int sx_gemm_plan(int M, int Nf, int K, int dual, int splits_req, int* bn_out, int* splits_out,
                            long long* ws_floats_out) {
  if (M <= 0 || Nf <= 0 || K <= 0 || (K % 64) != 0)
    return arg_error("sx_gemm: need M,N > 0 and K a positive multiple of 64 (M=%d N=%d K=%d)", M, Nf, K);
  const int bn = pick_bn(M, dual ? 128 : bn_cap_single());
  const int tiles_t = (M + bn - 1) / bn;
  const int tiles_f = (Nf + 127) / 128;
  const int kb_total = K / 64;
  int splits = splits_req;
  if (splits <= 0) {
    const int units = tiles_t * tiles_f;
    splits = 1;
    // weight-streaming shapes: split K until the grid covers the SMs,
    // keeping at least 8 k-blocks (512 of K) per split.
    while (units * splits < (kNumSMs * 3) / 4 && kb_total / (splits * 2) >= 8) splits *= 2;
  }
  if (splits > kb_total) splits = kb_total;
  const int kps = (kb_total + splits - 1) / splits;
  splits = (kb_total + kps - 1) / kps;
  *bn_out = bn;
  *splits_out = splits;
  *ws_floats_out = splits > 1 ? (long long)splits * (dual ? 2 : 1) * M * (long long)Nf : 0;
  return SX_OK;
}

extern "C" int sx_gemm_bf16(const void* W, const void* W2, const void* X, void* out, float* ws,
                            long long ws_floats, int M, int Nf, int K, long long ldo, int epi, int splits_req,
                            cudaStream_t stream) {
  const int dual = W2 != nullptr;
  if (dual != (epi == SX_EPI_SWIGLU_BF16)) return arg_error("sx_gemm: SWIGLU epilogue needs W2 and vice versa");
  if (epi < 0 || epi > SX_EPI_SWIGLU_BF16) return arg_error("sx_gemm: bad epilogue %d", epi);
  if (ldo < Nf) return arg_error("sx_gemm: ldo (%lld) < N (%d)", ldo, Nf);
  int bn, splits;
  long long need;
  int st = sx_gemm_plan(M, Nf, K, dual, splits_req, &bn, &splits, &need);
  if (st) return st;
  if (need > 0 && (ws == nullptr || ws_floats < need))
    return arg_error("sx_gemm: split-K workspace needs %lld floats, got %lld", need, ws_floats);

  // CTA-pair (cta_group::2) path for the compute-bound shapes
  const bool pair = splits == 1 && Nf >= 256 && (g_pair_mode == 2 || (g_pair_mode == 0 && M >= 256));
  if (pair) bn = (pick_bn(M, dual ? 128 : bn_cap_single()) + 31) / 32 * 32;

  CUtensorMap ma, ma2, mb;
  if ((st = make_tmap_bf16_kmajor(&ma, W, Nf, K, K, 128))) return st;
  if ((st = make_tmap_bf16_kmajor(&ma2, dual ? W2 : W, Nf, K, K, 128))) return st;
  if ((st = make_tmap_bf16_kmajor(&mb, X, M, K, K, pair ? bn / 2 : bn))) return st;

  if (pair) {
    GemmArgs g{};
    g.M = M;
    g.Nf = Nf;
    g.K = K;
    g.BN = bn;
    g.tiles_f = (Nf + 255) / 256;
    g.tiles_t = (M + bn - 1) / bn;
    g.kb_total = K / 64;
    g.splits = 1;
    g.kb_per_split = g.kb_total;
    g.units = g.tiles_f * g.tiles_t;
    g.epi = epi;
    g.dual = dual;
    g.a_bytes = 128 * 64 * 2;
    g.b_bytes = (bn / 2) * 64 * 2;
    g.stage_bytes = (dual ? 2 : 1) * g.a_bytes + g.b_bytes;
    g.stages = (227 * 1024 - 1024 - 256) / (int)g.stage_bytes;
    if (g.stages > max_stages()) g.stages = max_stages();
    g.acc_cols = bn * (dual ? 2 : 1);
    g.acc_stages = (2 * g.acc_cols <= 512) ? 2 : 1;
    uint32_t cols = 32;
    while (cols < g.acc_cols * (uint32_t)g.acc_stages) cols <<= 1;
    g.tmem_cols = cols;
    g.out = out;
    g.ldo = ldo;
    g.ws = nullptr;
    const size_t smem = 1024 + (size_t)g.stages * g.stage_bytes + (2 * g.stages + 4) * 8 + 16;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(gemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr2 = true;
    }
    const int pairs = g.units < kNumSMs / 2 ? g.units : kNumSMs / 2;
    gemm_tc2_kernel<<<2 * pairs, kGemmThreads, smem, stream>>>(ma, ma2, mb, g);
    SX_CHECK_LAUNCH("gemm_tc2_kernel");
    return SX_OK;
  }

  GemmArgs g{};
  g.M = M;
  g.Nf = Nf;
  g.K = K;
  g.BN = bn;
  g.tiles_f = (Nf + 127) / 128;
  g.tiles_t = (M + bn - 1) / bn;
  g.kb_total = K / 64;
  g.splits = splits;
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  g.units = g.tiles_f * g.tiles_t * splits;
  g.epi = epi;
  g.dual = dual;
  g.a_bytes = 128 * 64 * 2;
  g.b_bytes = bn * 64 * 2;
  g.stage_bytes = (dual ? 2 : 1) * g.a_bytes + g.b_bytes;
  const int smem_budget = 227 * 1024 - 1024 - 256;
  g.stages = smem_budget / (int)g.stage_bytes;
  if (g.stages > max_stages()) g.stages = max_stages();
  g.acc_cols = bn * (dual ? 2 : 1);
  g.acc_stages = (2 * g.acc_cols <= 512) ? 2 : 1;
  uint32_t need_cols = g.acc_cols * g.acc_stages;
  uint32_t cols = 32;
  while (cols < need_cols) cols <<= 1;
  g.tmem_cols = cols;
  g.out = out;
  g.ldo = ldo;
  g.ws = ws;

  const size_t smem = 1024 + (size_t)g.stages * g.stage_bytes + (2 * g.stages + 4) * 8 + 16;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  int grid = g.units < kNumSMs ? g.units : kNumSMs;
  gemm_tc_kernel<<<grid, kGemmThreads, smem, stream>>>(ma, ma2, mb, g);
  SX_CHECK_LAUNCH("gemm_tc_kernel");
  if (splits > 1) {
    long long total = (long long)M * Nf;
    int blocks = (int)((total + 255) / 256);
    if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(ws, out, ldo, M, Nf, splits, epi, dual);
    SX_CHECK_LAUNCH("splitk_reduce_kernel");
  }
  return SX_OK;
}
