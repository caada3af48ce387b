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
// Structure: persistent, warp-specialised, one CTA (or CTA pair) per SM.
//   warp 0      TMA producer   (weights + token tiles, 128B swizzle, mbarrier ring;
//                               two 64-wide k-blocks per stage, KPB = 2)
//   warp 1      TMEM allocator + the tcgen05.mma issuer (warp-uniform loop, elect.sync)
//   warps 2..5  epilogue       (tcgen05.ld -> registers -> fused epilogue -> global)
// Accumulators are double-buffered in TMEM when they fit so the epilogue of one
// tile overlaps the main loop of the next.
//
// Tile shapes (template CG): CG = 2 is a CTA pair (cta_group::2, a 2-CTA
// cluster): 256 weight rows per tile, each CTA stages half the token tile, one
// MMA issued by the even CTA covers both -- half the token-operand traffic per
// weight row, used for tree passes (128..~1k tokens). CG = 1 is a single CTA with
// 16..256-token tiles for thin draft batches and the one-token root / chain
// steps (optionally in 2/4-CTA clusters that multicast the token tile, opt-in).
// `make_plan` picks CG, the token-tile width (a wave-cost search over widths for
// pair shapes) and the schedule.
//
// Scheduling (`SegIter`): 0 whole tiles round-robin; 1 STREAM-K, the (tile,
// k-block) space cut into one contiguous range per CTA; 2 whole-tile waves and
// a K-split tail; 3 whole-tile waves and a stream-K tail (explicit request
// only). A tile split across CTAs is finished by its "owner" (the CTA holding
// its first k-block); the others publish fp32 partials + a flag and the owner
// adds them in a fixed order -- deterministic, no atomics on data.
//
// Epilogues (`epilogue_store`): bf16, fp32 (logits), fp32 residual add,
// SwiGLU over an interleaved gate/up weight (SX_EPI_SWIGLU_IL: the up rows of
// each 16-row group are exchanged through shared memory), the legacy dual-
// accumulator SwiGLU (DUAL), reduce-scatter into peer inboxes over NVLink
// (SX_EPI_RS_BF16) and QKV with RoPE applied and K / V scattered into the cache
// (SX_EPI_QKV_ROPE). Stores go through a 16-token x 128-feature fp32 smem tile
// so each thread writes 16-byte runs along the feature dimension.
#include "capi_util.h"
#include "common.cuh"
#include "gemv.h"
#include "specexec_b200.h"

namespace sx {

struct GemmArgs {
  int M, Nf, K;
  int BN;
  int tiles_f, tiles_t, kb_total, tiles;  // kb_total in units of BK = 64 * kpb
  int streamk;      // 0: whole tiles round-robin, 1: stream-K ranges, 2: whole-tile waves + split tail
  long long work;   // tiles * kb_total
  int ctas;         // scheduling units (CTAs, or CTA pairs when cta_group::2)
  int dp_rounds;    // mode 2: whole-tile rounds before the tail
  int tail_tiles;   // mode 2: tiles left for the split tail
  int tail_splits;  // mode 2: K-splits per tail tile
  int epi, stages;
  uint32_t stage_bytes, a_bytes, b_bytes;  // a/b: one 64-wide swizzle atom of the A / B tile (this CTA's rows)
  uint32_t acc_cols;  // TMEM columns per accumulator buffer
  int acc_stages;
  uint32_t tmem_cols;
  void* out;
  long long ldo;
  // SX_EPI_RS_BF16 (tensor-parallel row-parallel projections): out = device array
  // of `rs_world` peer inbox pointers; feature f goes to owner f / rs_slice, at
  // inbox[owner][rs_rank][t][f - owner * rs_slice] (bf16) -- the reduce-scatter
  // half of the all-reduce, written by the epilogue over NVLink as tiles finish
  int rs_rank, rs_world, rs_slice;
  int vec_store;  // 1: output rows 16-B aligned -> smem-transposed epilogue with 16-B stores
  int mc;         // single-CTA tiles: cluster of mc CTAs on consecutive weight tiles sharing one token
                  // tile, each loading 1/mc of it with TMA multicast (1 = off)
  uint32_t b_full_bytes;  // one 64-wide atom of the whole token tile (mc > 1)
  // SX_EPI_QKV_ROPE: rows = [q heads | k heads | v heads] x 128; each 128-row tile is one head
  const int* rope_pos;
  const int* rope_slot;
  int rope_pos_base, rope_slot_base, rope_H, rope_KVH;
  const float* rope_cos;
  const float* rope_sin;
  __nv_bfloat16* rope_q;
  __nv_bfloat16* rope_kc;
  __nv_bfloat16* rope_vc;
  long long rope_slots;
  int* flags;      // stream-K partial-ready flags [ctas * CG]
  float* part;     // stream-K partials [ctas * CG][dual?2:1][BN][128]
  int debug_no_tma;  // measurement builds (-DSX_GEMM_MEASURE_MMA_ONLY) + SX_GEMM_DEBUG=1: skip TMA after the first ring fill (MMA-rate measurement only)
};

constexpr int kGemmThreads = 192;
constexpr int kFlagFloats = 1024;  // workspace prefix reserved for the stream-K flags

SX_DEV float silu(float x) { return x / (1.0f + __expf(-x)); }
SX_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---- work segments: (tile, kb0, kb1) in processing order for unit c ---------
struct SegIter {
  long long pos, end;
  int t, step, c, r;
  int mode;
  bool tail_done;
  SX_DEV SegIter(const GemmArgs& g, int unit) {
    mode = g.streamk;
    c = unit;
    r = 0;
    tail_done = false;
    if (mode == 1 || mode == 3) {  // (mode 3: the stream-K ranges of the tail, after the whole-tile rounds)
      pos = (g.work * c) / g.ctas;
      end = (g.work * (c + 1)) / g.ctas;
    } else {
      t = c;
      step = g.ctas;
    }
  }
  SX_DEV bool next(const GemmArgs& g, int& tile, int& kb0, int& kb1) {
    if (mode == 3) {
      if (r < g.dp_rounds) {  // whole tiles first
        tile = r * g.ctas + c;
        kb0 = 0;
        kb1 = g.kb_total;
        ++r;
        return true;
      }
      if (pos >= end) return false;
      tile = g.dp_rounds * g.ctas + (int)(pos / g.kb_total);
      kb0 = (int)(pos % g.kb_total);
      kb1 = (int)min((long long)g.kb_total, kb0 + (end - pos));
      pos += kb1 - kb0;
      return true;
    }
    if (mode == 1) {
      if (pos >= end) return false;
      tile = (int)(pos / g.kb_total);
      kb0 = (int)(pos % g.kb_total);
      kb1 = (int)min((long long)g.kb_total, kb0 + (end - pos));
      pos += kb1 - kb0;
      return true;
    }
    if (mode == 2) {
      if (r < g.dp_rounds) {  // whole tiles: in round r the units cover tiles r*P .. r*P+P-1
        tile = r * g.ctas + c;
        kb0 = 0;
        kb1 = g.kb_total;
        ++r;
        return true;
      }
      if (tail_done || c >= g.tail_tiles * g.tail_splits) return false;
      tail_done = true;  // one tail item per unit; all items run concurrently
      const int j = c % g.tail_tiles, s = c / g.tail_tiles;
      tile = g.dp_rounds * g.ctas + j;
      kb0 = (int)((long long)g.kb_total * s / g.tail_splits);
      kb1 = (int)((long long)g.kb_total * (s + 1) / g.tail_splits);
      return true;
    }
    if (t >= g.tiles) return false;
    tile = t;
    kb0 = 0;
    kb1 = g.kb_total;
    t += step;
    return true;
  }
};

SX_DEV long long sk_start(const GemmArgs& g, int c) { return (g.work * c) / g.ctas; }
// unit whose range contains linear k-block k
SX_DEV int sk_unit_of(const GemmArgs& g, long long k) {
  int c = (int)((k * g.ctas) / g.work);
  while (c + 1 < g.ctas && sk_start(g, c + 1) <= k) ++c;
  while (c > 0 && sk_start(g, c) > k) --c;
  return c;
}

SX_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
SX_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SX_DEV void st_release(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

// Final epilogue of one 16-column chunk (values already summed over K).
// xs: 16 x 128 fp32 smem tile (8 KB). Vector path: the 4 epilogue warps write
// their rows (thread = feature, 16 tokens each) into xs[token][feature], then
// every thread stores 16-byte runs of consecutive features of one token row
// (8 bf16 / 4 fp32) instead of 16 scattered 2-4 byte stores; SWIGLU_IL reads
// gate (rows 0..63) and up (rows 64..127) of the same 64 features from xs.
SX_DEV void epilogue_store(const GemmArgs& g, const float (&v)[16], const float (&v2)[16], int f, int fl, bool fok,
                           int t0, float* xs) {
  const int fbase = f - fl;  // first feature (weight row) of this CTA's 128-row tile
  if (g.vec_store && (g.epi == SX_EPI_BF16 || g.epi == SX_EPI_F32 || g.epi == SX_EPI_SWIGLU_IL ||
                      g.epi == SX_EPI_RS_BF16 || g.epi == SX_EPI_QKV_ROPE)) {
#pragma unroll
    for (int j = 0; j < 16; ++j) xs[j * 128 + fl] = v[j];
    epi_bar();
    const int tid = fl;  // 0..127
    if (g.epi == SX_EPI_QKV_ROPE) {
      // this tile = head hh for 16 tokens; thread: token j, dims d0..d0+7 and their +64 partners
      const int hh = fbase >> 7;
      const int j = tid >> 3, d0 = (tid & 7) * 8;
      const int t = t0 + j;
      if (t < g.M && fbase < g.Nf) {
        const float* x = xs + j * 128;
        const long long sl = g.rope_slot_base + (g.rope_slot ? g.rope_slot[t] : t);
        __nv_bfloat16* dst;
        if (hh < g.rope_H)
          dst = g.rope_q + ((long long)t * g.rope_H + hh) * 128;
        else if (hh < g.rope_H + g.rope_KVH)
          dst = g.rope_kc + ((long long)(hh - g.rope_H) * g.rope_slots + sl) * 128;
        else
          dst = g.rope_vc + ((long long)(hh - g.rope_H - g.rope_KVH) * g.rope_slots + sl) * 128;
        float lo[8], hi[8];
        if (hh < g.rope_H + g.rope_KVH) {  // rotate-half RoPE (HF convention) at position p
          const long long p = g.rope_pos_base + (g.rope_pos ? g.rope_pos[t] : t);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float c = g.rope_cos[p * 64 + d0 + i], sn = g.rope_sin[p * 64 + d0 + i];
            const float x0 = x[d0 + i], x1 = x[d0 + 64 + i];
            lo[i] = x0 * c - x1 * sn;
            hi[i] = x1 * c + x0 * sn;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            lo[i] = x[d0 + i];
            hi[i] = x[d0 + 64 + i];
          }
        }
        uint4 a, b;
        a.x = pack_bf16x2(lo[0], lo[1]);
        a.y = pack_bf16x2(lo[2], lo[3]);
        a.z = pack_bf16x2(lo[4], lo[5]);
        a.w = pack_bf16x2(lo[6], lo[7]);
        b.x = pack_bf16x2(hi[0], hi[1]);
        b.y = pack_bf16x2(hi[2], hi[3]);
        b.z = pack_bf16x2(hi[4], hi[5]);
        b.w = pack_bf16x2(hi[6], hi[7]);
        *reinterpret_cast<uint4*>(dst + d0) = a;
        *reinterpret_cast<uint4*>(dst + d0 + 64) = b;
      }
    } else if (g.epi == SX_EPI_BF16 || g.epi == SX_EPI_RS_BF16) {
      // 16 tokens x 16 groups of 8 features = 256 items, 2 per thread
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int item = tid + it * 128, j = item >> 4, grp = item & 15;
        const int t = t0 + j, f0 = fbase + grp * 8;
        if (t < g.M) {
          const float* src = xs + j * 128 + grp * 8;
          __nv_bfloat16* o;
          if (g.epi == SX_EPI_RS_BF16) {  // owner's inbox over peer memory: 16-B stores into its slice
            const int owner = f0 / g.rs_slice;
            o = reinterpret_cast<__nv_bfloat16* const*>(g.out)[owner] +
                ((long long)g.rs_rank * g.M + t) * g.rs_slice + (f0 - owner * g.rs_slice);
          } else {
            o = reinterpret_cast<__nv_bfloat16*>(g.out) + (long long)t * g.ldo + f0;
          }
          if (f0 + 8 <= g.Nf) {
            uint4 pk;
            pk.x = pack_bf16x2(src[0], src[1]);
            pk.y = pack_bf16x2(src[2], src[3]);
            pk.z = pack_bf16x2(src[4], src[5]);
            pk.w = pack_bf16x2(src[6], src[7]);
            *reinterpret_cast<uint4*>(o) = pk;
          } else {
            for (int e = 0; e < 8 && f0 + e < g.Nf; ++e) o[e] = __float2bfloat16(src[e]);
          }
        }
      }
    } else if (g.epi == SX_EPI_F32) {
      // 16 tokens x 32 groups of 4 features = 512 items, 4 per thread
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int item = tid + it * 128, j = item >> 5, grp = item & 31;
        const int t = t0 + j, f0 = fbase + grp * 4;
        if (t < g.M) {
          const float4 val = *reinterpret_cast<const float4*>(xs + j * 128 + grp * 4);
          float* o = reinterpret_cast<float*>(g.out) + (long long)t * g.ldo + f0;
          if (f0 + 4 <= g.Nf) {
            *reinterpret_cast<float4*>(o) = val;
          } else {
            const float vv[4] = {val.x, val.y, val.z, val.w};
            for (int e = 0; e < 4 && f0 + e < g.Nf; ++e) o[e] = vv[e];
          }
        }
      }
    } else {  // SWIGLU_IL: 16 tokens x 8 groups of 8 output features = 128 items
      const int j = tid >> 3, grp = tid & 7;
      const int t = t0 + j;
      if (t < g.M && fbase < g.Nf) {  // a pair's second CTA may hold rows past N
        const float* gs = xs + j * 128 + grp * 8;
        const float* us = gs + 64;
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out) + (long long)t * g.ldo + (fbase >> 1) + grp * 8;
        uint4 pk;
        pk.x = pack_bf16x2(silu(gs[0]) * us[0], silu(gs[1]) * us[1]);
        pk.y = pack_bf16x2(silu(gs[2]) * us[2], silu(gs[3]) * us[3]);
        pk.z = pack_bf16x2(silu(gs[4]) * us[4], silu(gs[5]) * us[5]);
        pk.w = pack_bf16x2(silu(gs[6]) * us[6], silu(gs[7]) * us[7]);
        *reinterpret_cast<uint4*>(o) = pk;
      }
    }
    epi_bar();  // xs is rewritten by the next chunk
    return;
  }
  if (g.epi == SX_EPI_BF16) {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (t0 + j < g.M && fok) o[(long long)(t0 + j) * g.ldo + f] = __float2bfloat16(v[j]);
  } else if (g.epi == SX_EPI_F32) {
    float* o = reinterpret_cast<float*>(g.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (t0 + j < g.M && fok) o[(long long)(t0 + j) * g.ldo + f] = v[j];
  } else if (g.epi == SX_EPI_ADD_F32) {
    float* o = reinterpret_cast<float*>(g.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (t0 + j < g.M && fok) o[(long long)(t0 + j) * g.ldo + f] += v[j];
  } else if (g.epi == SX_EPI_RS_BF16) {
    if (fok) {
      __nv_bfloat16* const* peers = reinterpret_cast<__nv_bfloat16* const*>(g.out);
      const int owner = f / g.rs_slice;
      __nv_bfloat16* o = peers[owner] + (long long)g.rs_rank * g.M * g.rs_slice + (f - owner * g.rs_slice);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (t0 + j < g.M) o[(long long)(t0 + j) * g.rs_slice] = __float2bfloat16(v[j]);
    }
  } else if (g.epi == SX_EPI_SWIGLU_IL) {
    const int r = fl & 63;
    if (fl >= 64) {
#pragma unroll
      for (int j = 0; j < 16; ++j) xs[j * 64 + r] = v[j];
    }
    epi_bar();
    if (fl < 64) {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out);
      const int fo = (fbase >> 1) + r;  // tile rows 128j.. -> output features 64j..
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (t0 + j < g.M && fok) o[(long long)(t0 + j) * g.ldo + fo] = __float2bfloat16(silu(v[j]) * xs[j * 64 + r]);
    }
    epi_bar();
  } else {  // SX_EPI_SWIGLU_BF16
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (t0 + j < g.M && fok) o[(long long)(t0 + j) * g.ldo + f] = __float2bfloat16(silu(v[j]) * v2[j]);
  }
}

// TMEM accumulator (this thread's lane = feature f, BN token columns) -> global.
//   mode 0: whole tile          -> final epilogue
//   mode 1: helper segment      -> fp32 partial in slot `slot`, then publish flag
//   mode 2: owner of split tile -> add the partials of slots h0, h0+hs, ... (hn of them) in order
template <bool DUAL>
SX_DEV void epilogue_seg(const GemmArgs& g, uint32_t tbase, int f, int fl, bool fok, int tt, int mode, int slot,
                         int h0, int hs, int hn, float* xs) {
  const long long pstride = (long long)(DUAL ? 2 : 1) * g.BN * 128;
  if (mode == 2) {
    if (threadIdx.x == 64)
      for (int i = 0; i < hn; ++i) {
        while (ld_acquire(&g.flags[h0 + i * hs]) == 0) {
        }
      }
    epi_bar();
  }
  for (int c = 0; c < g.BN; c += 16) {
    uint32_t r[16];
    uint32_t r2[16];
    tmem_ld16(tbase + c, r);
    if (DUAL) tmem_ld16(tbase + g.BN + c, r2);
    tmem_ld_wait();
    float v[16], v2[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = __uint_as_float(r[j]);
      v2[j] = DUAL ? __uint_as_float(r2[j]) : 0.f;
    }
    // partial layout per slot: [token/4][feature][4] floats -> one float4 per 4 tokens
    if (mode == 1) {
      float4* p = reinterpret_cast<float4*>(g.part + slot * pstride) + (long long)(c >> 2) * 128 + fl;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        p[q * 128] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if (DUAL)
          p[(long long)g.BN * 32 + q * 128] = make_float4(v2[4 * q], v2[4 * q + 1], v2[4 * q + 2], v2[4 * q + 3]);
      }
      continue;
    }
    if (mode == 2) {
      for (int i = 0; i < hn; ++i) {
        const float4* p = reinterpret_cast<const float4*>(g.part + (h0 + i * hs) * pstride) +
                          (long long)(c >> 2) * 128 + fl;
        float4 a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[q] = __ldcg(p + q * 128);
          if (DUAL) b[q] = __ldcg(p + (long long)g.BN * 32 + q * 128);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[4 * q] += a[q].x;
          v[4 * q + 1] += a[q].y;
          v[4 * q + 2] += a[q].z;
          v[4 * q + 3] += a[q].w;
          if (DUAL) {
            v2[4 * q] += b[q].x;
            v2[4 * q + 1] += b[q].y;
            v2[4 * q + 2] += b[q].z;
            v2[4 * q + 3] += b[q].w;
          }
        }
      }
    }
    epilogue_store(g, v, v2, f, fl, fok, tt * g.BN + c, xs);
  }
  if (mode == 1) {
    __threadfence();
    epi_bar();
    if (threadIdx.x == 64) st_release(&g.flags[slot], 1);
  } else if (mode == 2) {
    epi_bar();  // every thread finished reading the partials
    if (threadIdx.x == 64)
      for (int i = 0; i < hn; ++i) g.flags[h0 + i * hs] = 0;  // re-arm for the next launch / graph replay
  }
}

// ---- cta_group-dependent primitives -----------------------------------------
template <int CG>
SX_DEV void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint64_t pol) {
  if constexpr (CG == 1)
    tma_load_2d_hint(dst, map, bar, c0, c1, pol);
  else
    tma_load_2d_2sm(dst, map, bar, c0, c1, pol);
}
template <int CG>
SX_DEV void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1)
    tc_mma_bf16(d, a, b, idesc, acc);
  else
    tc_mma_bf16_2sm(d, a, b, idesc, acc);
}
template <int CG>
SX_DEV void commit(uint64_t* bar) {
  if constexpr (CG == 1)
    tc_commit(bar);
  else
    tc_commit_2sm_mc(bar, 0x3);
}

// One kernel for both MMA shapes:
//   CG = 1: one CTA per tile, M = 128 weight rows, BN tokens;
//   CG = 2: a CTA pair (cluster of 2, tcgen05 cta_group::2) per tile, M = 256
//           weight rows (128 per CTA), each CTA stages half of the BN token rows,
//           the leader issues the pair MMA -- half the B-operand smem traffic per SM.
// KPB = 64-wide k-blocks (swizzle atoms) per pipeline stage: 2 halves the
// mbarrier round trips (wait + commit) per MMA.
template <int CG, bool DUAL, int KPB>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB, const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms (same offset in both CTAs of a pair).
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + g.stages * g.stage_bytes);
  uint64_t* empty_bar = full_bar + g.stages;
  uint64_t* tfull_bar = empty_bar + g.stages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  float* xs = reinterpret_cast<float*>(smem + g.stages * g.stage_bytes + 1024);  // epilogue tile, 8 KB

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int MC = CG == 1 ? g.mc : 1;
  const uint32_t mrank = MC > 1 ? cluster_ctarank() : 0u;  // position in the multicast cluster
  const int unit = blockIdx.x / (CG * MC);

  griddep_launch_dependents();  // a PDL-launched successor may set up while this grid runs
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    if (DUAL) tma_prefetch_desc(&mapA2);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MC);  // multicast: a stage is free once every CTA's MMA released it
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4 * CG);  // 4 epilogue warps per CTA (pair: both CTAs arrive at the leader)
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 1)
      tmem_alloc(tmem_base_smem, g.tmem_cols);
    else
      tmem_alloc_2sm(tmem_base_smem, g.tmem_cols);
  }
  tc_fence_before();
  if (CG == 2 || MC > 1)
    cluster_sync();  // peers' barriers are initialised before any multicast / remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  const uint32_t a_off = (DUAL ? 2 : 1) * KPB * g.a_bytes;  // B atoms follow the A (and A2) atoms
  if (warp == 0) {
    // ---------------- TMA producer (warp-uniform loop, one elected lane issues) ----------------
    // weights: evict-first when a single token tile reads each weight tile once;
    // with several token tiles the sibling CTAs re-read it from L2 (evict-first
    // measured +60% DRAM re-reads on the 70B SwiGLU / down projections)
    const uint64_t pol_w = g.tiles_t == 1 ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_x = policy_evict_last();   // token tiles are re-read by every weight tile
    const int bhalf = g.BN / CG;
    {
      // Programmatic dependent launch: this grid may start while the previous
      // kernel drains. The weights do not depend on it -- warm L2 with the first
      // ring of weight boxes, then wait before touching its outputs (tokens).
      SegIter it0(g, unit);
      int tile, kb0, kb1;
      if (it0.next(g, tile, kb0, kb1) && elect_one()) {
        const int frow = ((tile / g.tiles_t) * MC + (int)mrank) * 128 * CG + (int)rank * 128;
        const int n = min(kb1 - kb0, g.stages);
        for (int kb = kb0; kb < kb0 + n; ++kb)
          for (int j = 0; j < KPB; ++j) {
            tma_prefetch_2d(&mapA, (kb * KPB + j) * 64, frow);
            if (DUAL) tma_prefetch_2d(&mapA2, (kb * KPB + j) * 64, frow);
          }
      }
      __syncwarp();
      griddep_wait();
    }
    int stage = 0;
    uint32_t phase = 0;
    int issued = 0;
    SegIter it(g, unit);
    int tile, kb0, kb1;
    const int bslice = g.BN / MC;  // token rows this CTA loads (and multicasts when MC > 1)
    while (it.next(g, tile, kb0, kb1)) {
      const int tt = tile % g.tiles_t;
      const int tf = (tile / g.tiles_t) * MC + (int)mrank;
      const int frow = tf * 128 * CG + (int)rank * 128;
      const int trow = tt * g.BN + (int)rank * bhalf + (int)mrank * bslice;
      for (int kb = kb0; kb < kb1; ++kb, ++issued) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * g.stage_bytes;
        if (elect_one()) {
          if (g.debug_no_tma && issued >= g.stages) {  // measurement mode: MMA on stale tiles
            if (rank == 0) mbar_arrive(&full_bar[stage]);
          } else {
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], CG * g.stage_bytes);
#pragma unroll
            for (int j = 0; j < KPB; ++j) {
              const int kc = (kb * KPB + j) * 64;
              tma_load<CG>(sa + j * g.a_bytes, &mapA, &full_bar[stage], kc, frow, pol_w);
              if (DUAL) tma_load<CG>(sa + (KPB + j) * g.a_bytes, &mapA2, &full_bar[stage], kc, frow, pol_w);
              if (CG == 1 && MC > 1)  // my slice of the shared token tile, to every CTA of the cluster
                tma_load_2d_mc(sa + a_off + j * g.b_bytes + mrank * bslice * 128, &mapB, &full_bar[stage], kc, trow,
                               (uint16_t)((1u << MC) - 1), pol_x);
              else
                tma_load<CG>(sa + a_off + j * g.b_bytes, &mapB, &full_bar[stage], kc, trow, pol_x);
            }
          }
        }
        __syncwarp();
        if (++stage == g.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair: leader CTA only) ----------------
    // The whole warp walks the (warp-uniform) loop so descriptors and counters
    // live in uniform registers; one elected lane issues tcgen05.mma/commit.
    if (rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(128 * CG, g.BN);
      const uint64_t desc0 = smem_desc_k_sw128(smem);  // stage s adds s * stage_bytes >> 4
      const uint32_t a_atom = g.a_bytes >> 4, b_atom = g.b_bytes >> 4;
      const uint32_t b_off = a_off >> 4;
      const uint32_t stage_off = g.stage_bytes >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      SegIter it(g, unit);
      int tile, kb0, kb1;
      while (it.next(g, tile, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * g.acc_cols;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t ds = desc0 + (uint64_t)(stage * stage_off);
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < KPB; ++j) {
              const uint64_t da = ds + j * a_atom;
              const uint64_t db = ds + b_off + j * b_atom;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                // advance 16 bf16 = 32 B along K inside the swizzle atom (>>4 => +2)
                const uint32_t acc_flag = (kb > kb0 || j > 0 || k > 0) ? 1u : 0u;
                mma<CG>(d0, da + 2 * k, db + 2 * k, idesc, acc_flag);
                if (DUAL) mma<CG>(d0 + g.BN, da + KPB * a_atom + 2 * k, db + 2 * k, idesc, acc_flag);
              }
            }
            if (CG == 1 && MC > 1)
              tc_commit_mc(&empty_bar[stage], (uint16_t)((1u << MC) - 1));  // release the stage in every CTA
            else
              commit<CG>(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == g.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) commit<CG>(&tfull_bar[acc]);
        __syncwarp();
        if (++acc == g.acc_stages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    griddep_wait();  // outputs may still be read by the previous kernel
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int fl = quarter * 32 + lane;
    const int slot = unit * CG + (int)rank;  // this CTA's partial slot / flag
    int acc = 0;
    uint32_t acc_phase = 0;
    SegIter it(g, unit);
    int tile, kb0, kb1;
    while (it.next(g, tile, kb0, kb1)) {
      const int tt = tile % g.tiles_t;
      const int tf = (tile / g.tiles_t) * MC + (int)mrank;
      const int f = tf * 128 * CG + (int)rank * 128 + fl;
      const bool fok = f < g.Nf;
      int mode = 0, h0 = 0, hs = 1, hn = 0;
      if (kb0 > 0) {
        mode = 1;  // helper: publishes a partial for the tile's owner
      } else if (kb1 < g.kb_total) {
        mode = 2;  // owner: the rest of the tile is summed by other units (same rank)
        if (g.streamk == 1 || g.streamk == 3) {
          const long long t_lin = g.streamk == 3 ? tile - (long long)g.dp_rounds * g.ctas : tile;
          h0 = (unit + 1) * CG + (int)rank;
          hs = CG;
          hn = sk_unit_of(g, t_lin * g.kb_total + g.kb_total - 1) - unit;
        } else {
          h0 = (unit + g.tail_tiles) * CG + (int)rank;
          hs = g.tail_tiles * CG;
          hn = g.tail_splits - 1;
        }
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * g.acc_cols;
      epilogue_seg<DUAL>(g, tbase, f, fl, fok, tt, mode, slot, h0, hs, hn, xs);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1)
          mbar_arrive(&tempty_bar[acc]);
        else
          mbar_arrive_remote(&tempty_bar[acc], 0);
      }
      if (++acc == g.acc_stages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CG == 2 || MC > 1) cluster_sync();  // no CTA leaves while peers may still multicast / arrive into it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      tmem_dealloc(tmem_base, g.tmem_cols);
    else
      tmem_dealloc_2sm(tmem_base, g.tmem_cols);
  }
}

// 0 = auto (pair when the tree pass has >= 256 tokens), 1 = single-CTA only, 2 = pair whenever legal.
static int g_pair_mode = getenv("SX_GEMM_PAIR_MODE") ? atoi(getenv("SX_GEMM_PAIR_MODE")) : 0;  // A/B knob
// programmatic dependent launch of the GEMM (SX_GEMM_PDL=0 disables): the weight
// ring prefetch and the CTA prologue overlap the previous kernel's tail. Round 1
// measured no change (156.4 vs 156.2 ms); round 2, six alternating C2 runs each
// (profiles/r2/gemm_pdl_ab.txt): 147.2 vs 148.0 ms, 1229 vs 1224 TFLOP/s
static const int g_pdl = getenv("SX_GEMM_PDL") ? atoi(getenv("SX_GEMM_PDL")) : 1;

// tuning overrides (read once): SX_GEMM_BN_CAP (token-tile cap), SX_GEMM_STAGES (max pipeline depth),
// SX_GEMM_KPB (64-wide k-blocks per stage; 0 = auto)
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
static int kpb_req() {
  static int v = env_int("SX_GEMM_KPB", 0);
  return v;
}

static int pick_bn(int M, int cap) {
  int tiles = (M + cap - 1) / cap;
  int bn = (M + tiles - 1) / tiles;
  bn = (bn + 15) / 16 * 16;
  if (bn < 16) bn = 16;
  return bn;
}

struct Plan {
  int cg, mc, kpb, bn, tiles_f, tiles_t, tiles, kb_total, ctas, streamk;
  int dp_rounds, tail_tiles, tail_splits;
  int stages;
  uint32_t a_bytes, b_bytes, stage_bytes;
  long long ws_floats;
};

constexpr int kSmemBudget = 227 * 1024 - 1024 - 1024 - 8192;  // align pad, barriers, epilogue tile

// Returns the token-tile cap to use with CTA-pair tiles, or 0 for single-CTA tiles.
static int pair_cap(int M, int Nf, int dual, int cg_req) {
  const int cap = dual ? 128 : bn_cap_single();
  if (Nf < 256) return 0;
  const int mode = cg_req ? cg_req : g_pair_mode;
  if (mode == 1) return 0;
  if (mode == 2) return cap;
  // auto: pair tiles halve the B-operand smem traffic per SM; take them when they
  // still give >= 1.5 waves over the 74 pairs -- with the widest token tile for
  // the tree pass (hundreds of tokens), or with 128-token tiles for a batch of
  // 128-511 tokens (7B SwiGLU at M = 256: 97 -> 59 us vs narrow single-CTA
  // tiles, tools/gemm_plan_sweep.py). Thinner batches stay single-CTA.
  if (M < 128) return 0;
  auto tiles = [&](int bn) { return (long long)((Nf + 255) / 256) * ((M + bn - 1) / bn); };
  if (M >= 256 && tiles(pick_bn(M, cap)) * 2 >= 3 * (kNumSMs / 2)) return cap;
  // Wide token batches (the draft's 1024-token rounds) whose pair tiles fill >= 0.8
  // of one wave (7B o / down projections: 64 pair tiles): pairs win under the
  // power cap -- half the B-operand smem traffic per FLOP lifts the clock. In
  // isolation the two plans tie; in the C2 loop pairs-wherever-legal measured
  // 151.96 vs 153.46 ms over 7 alternating runs (profiles/r2/gemm_pair_ab.txt).
  if (M >= 512 && tiles(pick_bn(M, cap)) * 5 >= 4 * (kNumSMs / 2)) return cap;
  if (M < 512 && cap >= 128 && tiles(pick_bn(M, 128)) * 2 >= 3 * (kNumSMs / 2)) return 128;
  return 0;
}

// req = sched | cg << 4 | (bn_cap / 16) << 8 (a plan request; 0 = all auto):
// cg 1 = single-CTA tiles, 2 = CTA pair (else the sx_gemm_set_pair_mode policy);
// bn_cap = token-tile width cap (explicit: no narrowing);
// sched: 1 = whole tiles only, 2 = force stream-K ranges, 3 = force
// whole-tile waves + split tail; otherwise auto:
//  - whole tiles when the waves fill >= 95% of the units;
//  - else, with several token tiles per weight tile, whole-tile waves plus a
//    K-split tail (all tail items run together, so the token tiles of a weight
//    tile still read the same k-range at the same time and share it in L2);
//  - else (one token tile: every weight tile is read once anyway) stream-K.
static Plan make_plan(int M, int Nf, int K, int dual, int req) {
  Plan p{};
  const int sched_req = req & 15;
  const int cg_req = (req >> 4) & 3;
  const int bn_req = ((req >> 8) & 255) * 16;
  const int pcap = pair_cap(M, Nf, dual, cg_req);
  p.cg = pcap ? 2 : 1;
  const int P = kNumSMs / p.cg;  // scheduling units
  const int fr = 128 * p.cg;     // weight rows per tile
  int cap = pcap ? pcap : (dual ? 128 : bn_cap_single());
  if (bn_req > 0) cap = bn_req < cap ? bn_req : cap;
  p.bn = pick_bn(M, cap);
  p.tiles_f = (Nf + fr - 1) / fr;
  // CTA-pair tree-pass shapes: the token-tile width sets both the padding of
  // M = K+1 and how the tiles fill the 74 pairs; pick the width with the lowest
  // (rounds x width) over {auto, 176, 128} when it is >10% better (70B o-proj at
  // M = 1025: 160 tiles of 208 = 2.2 rounds -> 192 tiles of 176 = 2.6 rounds,
  // 118 -> 113 us; 70B down-proj (K = 28672): 208-wide tiles + split tail
  // 381-392 us -> 176-wide whole tiles 374-377 us, profiles/r1/plan_fine_down.jsonl;
  // neutral in the power-capped loop).
  if (p.cg == 2 && bn_req == 0 && !dual) {
    auto cost = [&](int bn) {
      const long long t = (long long)p.tiles_f * ((M + bn - 1) / bn);
      return (double)((t + P - 1) / P) * bn;
    };
    int best = p.bn;
    double best_cost = cost(p.bn);
    for (int c : {176, 128}) {
      const int bn = pick_bn(M, c < cap ? c : cap);
      if (cost(bn) < 0.9 * best_cost) {
        best = bn;
        best_cost = cost(bn);
      }
    }
    p.bn = best;
  }
  // Weight-streaming shapes with few weight tiles (e.g. a 4096-wide projection of
  // the draft = 32 tiles): a single SM's TMA pulls only ~40-50 GB/s, so use
  // narrower token tiles until ~120+ CTAs stream. The weight tile is shared by
  // the token tiles through L2, HBM traffic is unchanged.
  if (p.cg == 1 && bn_req == 0) {
    while (p.tiles_f * ((M + p.bn - 1) / p.bn) < 120 && p.bn > 32) {
      const int half = ((p.bn / 2) + 15) / 16 * 16;
      const int nb = pick_bn(M, half);
      if (p.tiles_f * ((M + nb - 1) / nb) > kNumSMs) break;  // would spill into a second wave
      p.bn = nb;
    }
    // Thin token batches (draft rounds): when whole tiles fill the waves poorly,
    // narrower token tiles buy wave efficiency for extra L2 re-reads of the weight
    // tile (7B SwiGLU at M = 256: 172 tiles, 97 -> 69 us at BN 256 -> 64;
    // tools/gemm_plan_sweep.py). Stop at 80% or BN 64.
    auto wave_eff = [&](int bn) {
      const long long t = (long long)p.tiles_f * ((M + bn - 1) / bn);
      const long long w = (t + kNumSMs - 1) / kNumSMs;
      return (double)t / (double)(w * kNumSMs);
    };
    while (M <= 512 && p.bn > 64 && wave_eff(p.bn) < 0.8) {
      const int nb = pick_bn(M, ((p.bn / 2) + 15) / 16 * 16);
      if (nb >= p.bn) break;
      p.bn = nb;
    }
  }
  p.tiles_t = (M + p.bn - 1) / p.bn;
  p.tiles = p.tiles_f * p.tiles_t;
  p.a_bytes = 128 * 64 * 2;
  p.b_bytes = (uint32_t)(p.bn / p.cg) * 64 * 2;
  // k-blocks per stage: 2 when K allows and >= 3 such stages fit (deep enough to hide TMA latency)
  auto stage_bytes = [&](int kpb) { return (uint32_t)kpb * ((dual ? 2 : 1) * p.a_bytes + p.b_bytes); };
  int kpb = kpb_req();
  if (kpb != 1 && kpb != 2) kpb = (K % 128 == 0 && kSmemBudget / (int)stage_bytes(2) >= 3) ? 2 : 1;
  if (K % (64 * kpb) != 0) kpb = 1;
  p.kpb = kpb;
  p.stage_bytes = stage_bytes(kpb);
  p.stages = kSmemBudget / (int)p.stage_bytes;
  const int stage_cap = (max_stages() + kpb - 1) / kpb;
  if (p.stages > stage_cap) p.stages = stage_cap;
  p.kb_total = K / (64 * kpb);
  const int waves = (p.tiles + P - 1) / P;
  const double eff = (double)p.tiles / ((double)waves * P);
  int mode = 0;
  if (sched_req == 2 || sched_req == 3 || sched_req == 4) {
    mode = sched_req == 4 ? 2 : sched_req - 1;  // 4: force the stream-K tail (resolved below)
  } else if (sched_req != 1 && eff < 0.95) {
    // several token tiles: waves + K-split tail (keeps the weight tile shared in
    // L2). One token tile: stream-K pays off only for thin token tiles (M <= 64:
    // 34 -> 19 us on a 4096 x 4096 projection at M = 2, 216 -> 104 us at M = 64,
    // K = 32768, tools/gemm_sched_micro.py; at M = 128 / 256 whole tiles win on
    // every 7B draft projection, e.g. qkv 37 -> 32 us, tools/gemm_bench.py).
    if (p.tiles_t > 1)
      mode = 2;
    else if (M <= 64)
      mode = 1;
  }
  if (mode == 2) {
    p.dp_rounds = p.tiles / P;
    p.tail_tiles = p.tiles - p.dp_rounds * P;
    int s = p.tail_tiles > 0 ? P / p.tail_tiles : 1;
    // the owner's fixup (reading s-1 partial tiles) must stay small next to a
    // tail item: measured a loss at 21 64-wide k-blocks per item (o-proj), a gain
    // at 64+ -- so split only as far as items keep >= 48 k-blocks (e.g. the 70B
    // SwiGLU: 10 tail tiles of 128 k-blocks -> 2 splits, not 7)
    if (sched_req != 3) {
      const int s_fix = p.kb_total * kpb / 48;
      if (s > s_fix) s = s_fix;
    }
    if (s > p.kb_total) s = p.kb_total;
    if (s < 1) s = 1;
    p.tail_splits = s;
    if (p.tail_tiles == 0) {
      mode = 0;  // nothing to balance
    } else if (sched_req == 4) {
      mode = p.dp_rounds > 0 ? 3 : 1;  // forced stream-K tail (no whole rounds: plain stream-K)
    } else if (s == 1) {
      // more tail tiles than half the units: whole tiles. (A stream-K tail --
      // sched 4 -- balances it but measured slower: 70B qkv 129 -> 143 us, o 105 ->
      // 115 us, C2 149 -> 158 ms/iteration; the partial fixups cost more than the
      // idle tail.)
      mode = 0;
    }
  }
  p.streamk = mode;
  // TMA multicast of the token tile (single-CTA, whole tiles): a cluster of mc
  // CTAs on consecutive weight tiles loads 1/mc of the shared token tile each and
  // multicasts it, so the token operand is not re-read from L2 per weight tile.
  // Opt-in (mc_req 2 / 4): on the 7B draft shapes at M = 256 the lock-stepped
  // clusters measured slower than independent CTAs (qkv 41 -> 64 us, gate/up
  // 97 -> 114 us, tools/gemm_plan_sweep.py), so the planner does not pick it.
  p.mc = 1;
  {
    const int mc_req = (req >> 16) & 7;
    int mc = 1;
    if (mc_req >= 2) mc = mc_req;
    while (mc > 1 && ((p.bn / mc) % 8 != 0 || p.cg != 1 || mode != 0 || mc > p.tiles_f)) mc >>= 1;
    if (mc > 1) {
      p.mc = mc;
      p.tiles = ((p.tiles_f + mc - 1) / mc) * p.tiles_t;  // cluster (group) tiles
    }
  }
  if (mode == 1) {
    p.ctas = P;
    if ((long long)p.tiles * p.kb_total < p.ctas) p.ctas = (int)((long long)p.tiles * p.kb_total);
  } else if (mode == 2) {
    p.ctas = p.dp_rounds > 0 ? P : p.tail_tiles * p.tail_splits;
  } else if (mode == 3) {
    p.ctas = P;
  } else {
    const int units = P / p.mc;
    p.ctas = p.tiles < units ? p.tiles : units;
  }
  p.ws_floats = mode ? kFlagFloats + (long long)p.ctas * p.cg * (dual ? 2 : 1) * p.bn * 128 : 0;
  return p;
}

template <int CG, bool DUAL, int KPB>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& ma2, const CUtensorMap& mb, const GemmArgs& g,
                       size_t smem, cudaStream_t stream) {
  auto kern = gemm_tc_kernel<CG, DUAL, KPB>;
  if (int st = ensure_smem_attr((const void*)kern, 227 * 1024)) return st;
  cudaLaunchConfig_t cfg{};
  const int cl = CG * (CG == 1 ? g.mc : 1);  // cluster: CTA pair, or the multicast group
  cfg.gridDim = dim3(g.ctas * cl);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol.wait in the kernel)
  at[1].val.programmaticStreamSerializationAllowed = g_pdl;
  // split tiles: owners wait on their helpers' flags, so the grid (<= one CTA or
  // pair per SM) must be co-resident -- a cooperative launch guarantees it even
  // when another engine's kernels share the GPU
  at[2].id = cudaLaunchAttributeCooperative;
  at[2].val.cooperative = g.flags != nullptr ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 3;
  cudaLaunchKernelEx(&cfg, kern, ma, ma2, mb, g);
  SX_CHECK_LAUNCH("gemm_tc_kernel");
  return SX_OK;
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
  Plan p = make_plan(M, Nf, K, dual, splits_req);
  *bn_out = p.bn;
  *splits_out = p.streamk ? p.ctas : 1;  // >1: number of stream-K units
  *ws_floats_out = p.ws_floats;
  return SX_OK;
}

static int gemm_launch(const void* W, const void* W2, const void* X, void* out, float* ws, long long ws_floats, int M,
                       int Nf, int K, long long ldo, int epi, int splits_req, int rs_rank, int rs_world, int rs_slice,
                       cudaStream_t stream, const GemmArgs* rope = nullptr);

extern "C" int sx_gemm_qkv_rope(const void* W, const void* X, float* ws, long long ws_floats, int M, int H, int KVH,
                                int K, const int* pos, int pos_base, const int* slot, int slot_base, const float* cos_t,
                                const float* sin_t, void* q, void* kcache, void* vcache, long long slots,
                                int splits_req, cudaStream_t stream) {
  if (H <= 0 || KVH <= 0) return arg_error("sx_gemm_qkv_rope: H, KVH must be > 0");
  if (!q || !kcache || !vcache || !cos_t || !sin_t) return arg_error("sx_gemm_qkv_rope: NULL output / table");
  GemmArgs r{};
  r.rope_pos = pos;
  r.rope_slot = slot;
  r.rope_pos_base = pos_base;
  r.rope_slot_base = slot_base;
  r.rope_H = H;
  r.rope_KVH = KVH;
  r.rope_cos = cos_t;
  r.rope_sin = sin_t;
  r.rope_q = reinterpret_cast<__nv_bfloat16*>(q);
  r.rope_kc = reinterpret_cast<__nv_bfloat16*>(kcache);
  r.rope_vc = reinterpret_cast<__nv_bfloat16*>(vcache);
  r.rope_slots = slots;
  const int Nf = (H + 2 * KVH) * 128;
  return gemm_launch(W, nullptr, X, q, ws, ws_floats, M, Nf, K, Nf, SX_EPI_QKV_ROPE, splits_req, 0, 1, Nf, stream, &r);
}

extern "C" int sx_gemm_bf16_rs(const void* W, const void* X, void* const* peer_inbox, int rank, int world, float* ws,
                               long long ws_floats, int M, int Nf, int K, int splits_req, cudaStream_t stream) {
  if (world < 1 || rank < 0 || rank >= world) return arg_error("sx_gemm_rs: bad rank %d / world %d", rank, world);
  if (Nf % world != 0 || (Nf / world) % 128 != 0)
    return arg_error("sx_gemm_rs: N=%d must split into %d slices of a multiple of 128", Nf, world);
  if (peer_inbox == nullptr) return arg_error("sx_gemm_rs: peer inbox table is NULL");
  return gemm_launch(W, nullptr, X, (void*)peer_inbox, ws, ws_floats, M, Nf, K, Nf, SX_EPI_RS_BF16, splits_req, rank,
                     world, Nf / world, stream);
}

extern "C" int sx_gemm_bf16(const void* W, const void* W2, const void* X, void* out, float* ws, long long ws_floats,
                            int M, int Nf, int K, long long ldo, int epi, int splits_req, cudaStream_t stream) {
  if (epi == SX_EPI_RS_BF16 || epi == SX_EPI_QKV_ROPE)
    return arg_error("sx_gemm: epilogue %d has its own entry point (sx_gemm_bf16_rs / sx_gemm_qkv_rope)", epi);
  return gemm_launch(W, W2, X, out, ws, ws_floats, M, Nf, K, ldo, epi, splits_req, 0, 1, Nf, stream);
}

static int gemm_launch(const void* W, const void* W2, const void* X, void* out, float* ws,
                       long long ws_floats, int M, int Nf, int K, long long ldo, int epi, int splits_req, int rs_rank,
                       int rs_world, int rs_slice, cudaStream_t stream, const GemmArgs* rope) {
  const int dual = W2 != nullptr;
  if (dual != (epi == SX_EPI_SWIGLU_BF16)) return arg_error("sx_gemm: SWIGLU epilogue needs W2 and vice versa");
  if (epi < 0 || epi > SX_EPI_QKV_ROPE) return arg_error("sx_gemm: bad epilogue %d", epi);
  if ((epi == SX_EPI_QKV_ROPE) != (rope != nullptr)) return arg_error("sx_gemm: QKV+RoPE epilogue via sx_gemm_qkv_rope");
  if (epi == SX_EPI_SWIGLU_IL && (Nf % 128) != 0)
    return arg_error("sx_gemm: interleaved SwiGLU needs N %% 128 == 0 (N=%d)", Nf);
  const int ncols = epi == SX_EPI_SWIGLU_IL ? Nf / 2 : Nf;
  if (ldo < ncols) return arg_error("sx_gemm: ldo (%lld) < output width (%d)", ldo, ncols);
  if (M <= 0 || Nf <= 0 || K <= 0 || (K % 64) != 0)
    return arg_error("sx_gemm: need M,N > 0 and K a positive multiple of 64 (M=%d N=%d K=%d)", M, Nf, K);
  int st;
  if (gemv_applies(M, epi, dual)) {  // 1..4 tokens: weight-streaming matrix-vector path (gemv.cu)
    GemvArgs v{};
    v.W = reinterpret_cast<const __nv_bfloat16*>(W);
    v.X = reinterpret_cast<const __nv_bfloat16*>(X);
    v.out = out;
    v.ldo = ldo;
    v.M = M;
    v.Nf = Nf;
    v.K = K;
    v.epi = epi;
    if (rope) {
      v.rope_pos = rope->rope_pos;
      v.rope_slot = rope->rope_slot;
      v.rope_pos_base = rope->rope_pos_base;
      v.rope_slot_base = rope->rope_slot_base;
      v.rope_H = rope->rope_H;
      v.rope_KVH = rope->rope_KVH;
      v.rope_cos = rope->rope_cos;
      v.rope_sin = rope->rope_sin;
      v.rope_q = rope->rope_q;
      v.rope_kc = rope->rope_kc;
      v.rope_vc = rope->rope_vc;
      v.rope_slots = rope->rope_slots;
    }
    return launch_gemv(v, stream);
  }
  Plan p = make_plan(M, Nf, K, dual, splits_req);
  if (p.ws_floats > 0 && (ws == nullptr || ws_floats < p.ws_floats))
    return arg_error("sx_gemm: stream-K workspace needs %lld floats, got %lld", p.ws_floats, ws_floats);
  CUtensorMap ma, ma2, mb;
  if ((st = make_tmap_bf16_kmajor(&ma, W, Nf, K, K, 128))) return st;
  if ((st = make_tmap_bf16_kmajor(&ma2, dual ? W2 : W, Nf, K, K, 128))) return st;
  if ((st = make_tmap_bf16_kmajor(&mb, X, M, K, K, p.bn / (p.cg * p.mc)))) return st;

  GemmArgs g{};
  g.M = M;
  g.Nf = Nf;
  g.K = K;
  g.BN = p.bn;
  g.tiles_f = p.tiles_f;
  g.tiles_t = p.tiles_t;
  g.kb_total = p.kb_total;
  g.tiles = p.tiles;
  g.streamk = p.streamk;
  // stream-K work: all (tile, k-block) pairs (mode 1) or only those of the tail (mode 3)
  g.work = (long long)(p.streamk == 3 ? p.tail_tiles : p.tiles) * p.kb_total;
  g.ctas = p.ctas;
  g.dp_rounds = p.dp_rounds;
  g.tail_tiles = p.tail_tiles;
  g.tail_splits = p.tail_splits;
  g.epi = epi;
  g.a_bytes = p.a_bytes;
  g.b_bytes = p.b_bytes;
  g.stage_bytes = p.stage_bytes;
  g.stages = p.stages;
  g.acc_cols = p.bn * (dual ? 2 : 1);
  g.acc_stages = (2 * g.acc_cols <= 512) ? 2 : 1;
  uint32_t cols = 32;
  while (cols < g.acc_cols * (uint32_t)g.acc_stages) cols <<= 1;
  g.tmem_cols = cols;
  g.out = out;
  g.ldo = ldo;
  g.vec_store = (ldo % 8 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) ? 1 : 0;
  if (epi == SX_EPI_RS_BF16) g.vec_store = (rs_slice % 128 == 0) ? 1 : 0;  // inbox rows are 16-B aligned slices
  if (rope) {
    g.rope_pos = rope->rope_pos;
    g.rope_slot = rope->rope_slot;
    g.rope_pos_base = rope->rope_pos_base;
    g.rope_slot_base = rope->rope_slot_base;
    g.rope_H = rope->rope_H;
    g.rope_KVH = rope->rope_KVH;
    g.rope_cos = rope->rope_cos;
    g.rope_sin = rope->rope_sin;
    g.rope_q = rope->rope_q;
    g.rope_kc = rope->rope_kc;
    g.rope_vc = rope->rope_vc;
    g.rope_slots = rope->rope_slots;
    g.vec_store = 1;  // head rows of 128 bf16, 16-B aligned
  }
  if (epi == SX_EPI_SWIGLU_IL && (Nf % 128)) g.vec_store = 0;
  g.mc = p.mc;
  g.rs_rank = rs_rank;
  g.rs_world = rs_world;
  g.rs_slice = rs_slice;
  g.flags = p.streamk ? reinterpret_cast<int*>(ws) : nullptr;
  g.part = p.streamk ? ws + kFlagFloats : nullptr;
#ifdef SX_GEMM_MEASURE_MMA_ONLY
  // measurement builds only (tools/gemm_probe.py: make MEASURE=1): MMA on stale
  // tiles after the first ring fill -- wrong results by design, never in the product
  static const int debug_no_tma = env_int("SX_GEMM_DEBUG", 0);
  g.debug_no_tma = debug_no_tma;
#else
  g.debug_no_tma = 0;
#endif

  const size_t smem = 1024 + (size_t)g.stages * g.stage_bytes + 1024 + 8192;
#define SX_GEMM_LAUNCH(CG, DU, KP) \
  if (p.cg == CG && dual == DU && p.kpb == KP) return launch_gemm<CG, DU, KP>(ma, ma2, mb, g, smem, stream);
  SX_GEMM_LAUNCH(1, 0, 1)
  SX_GEMM_LAUNCH(1, 0, 2)
  SX_GEMM_LAUNCH(1, 1, 1)
  SX_GEMM_LAUNCH(1, 1, 2)
  SX_GEMM_LAUNCH(2, 0, 1)
  SX_GEMM_LAUNCH(2, 0, 2)
  SX_GEMM_LAUNCH(2, 1, 1)
  SX_GEMM_LAUNCH(2, 1, 2)
#undef SX_GEMM_LAUNCH
  return arg_error("sx_gemm: no kernel for cg=%d dual=%d kpb=%d", p.cg, dual, p.kpb);
}
