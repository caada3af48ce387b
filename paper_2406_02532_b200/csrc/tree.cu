// KT1-KT3: stage-1 draft-tree construction on the GPU (build_sssp,
// pkg/src/speckit/tree.py:240-327).
//
// State kept in one device workspace (tree_layout.h):
//   materialized  : the <= K best candidates so far, SORTED by the reference key
//                   (nll asc, depth asc, path-lex asc) (tree.py:235-237, :270-278),
//                   double-buffered; each node carries its parent index, token,
//                   edge log-prob, draft-KV slot (if expanded) and its rank in
//                   path-lex order among same-depth nodes (`lex`).
//   batch         : the <= B nodes expanded by the next draft call (tree.py:282-295)
//   survivors     : this round's children whose key beats the threshold
//
// Key encoding: hi = bit pattern of nll (>= 0, so unsigned order == numeric
// order); lo = depth << 56 | lex(parent) << 32 | token. For two same-depth
// paths, lexicographic order == (lex rank of parent, token), so (hi, lo) is the
// reference's total order.
//
// Per round (one draft call):
//   scoring        : canonical float64 probabilities of every batch row (from
//                    fp32 logits, fp64 probabilities, or a warped row), edge =
//                    sx_log(p), nll = parent_nll - edge, keep key < threshold.
//                    fp32 logits (the Llama drafts) take the chunked persistent
//                    path: a max pass (one HBM read, exact row max + an fp32
//                    estimate that prefilters whole rows against the threshold)
//                    and one fused exact pass (canonical sums, then the edges of
//                    the candidates the estimate cannot rule out).
//   sx_tree_update : a cluster of kUpdCluster CTAs. When the survivors fit the
//                    sort buffer, CTA 0 sorts just them and merges them with the
//                    (already sorted) materialized list, and merges the lex
//                    order the same way. Otherwise (root round, floods): radix select (8-bit digits
//                    over the 128-bit key) of the K best of materialized U
//                    survivors: every CTA histograms its slice of the keys, the
//                    histograms are summed over distributed shared memory and
//                    the bin is found by a parallel scan in every CTA (identical
//                    result, no broadcast); the selected keys are gathered into
//                    CTA 0's shared memory. CTA 0 then bitonic-sorts them, remaps
//                    parents, recomputes lex ranks (sort by lo), sets the new
//                    threshold = K-th key and picks the next batch = first B
//                    unexpanded nodes with depth < D and key < threshold, their
//                    draft-KV slots and ancestor-slot lists.
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"
#include "sxmath.cuh"
#include "tree_layout.h"
#include "warp_rows.cuh"

#include <cooperative_groups.h>

namespace sx {

template <typename T>
SX_DEV T* at(uint8_t* ws, long long off) {
  return reinterpret_cast<T*>(ws + off);
}

SX_DEV unsigned long long make_lo(int depth, int plex, int token) {
  return ((unsigned long long)depth << 56) | ((unsigned long long)(unsigned)plex << 32) | (unsigned)token;
}
SX_DEV int lo_depth(unsigned long long lo) { return (int)(lo >> 56); }
SX_DEV int lo_token(unsigned long long lo) { return (int)(lo & 0xffffffffu); }

// Scoring kernels take the batch-row range [r0, r1) of this launch (r1 < 0: up to
// batch_n) -- the whole batch normally; slices of it when a round overflowed the
// survivor buffer and is re-run in parts (sx_tree_round_rows).
SX_DEV int rows_end(const TreeCtl* c, int r1) { return r1 < 0 ? c->batch_n : min(r1, c->batch_n); }

SX_DEV bool key_less(unsigned long long ah, unsigned long long al, unsigned long long bh, unsigned long long bl) {
  return ah < bh || (ah == bh && al < bl);
}

// --------------------------------------------------------------------------
__global__ void tree_begin_kernel(uint8_t* ws, TreeLayout L, int root_slot, int pad_slot) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  c->cur = 0;
  c->count = 0;
  c->has_thr = 0;
  c->rounds = 0;
  c->slot_next = root_slot + 1;
  c->batch_n = 1;
  c->n_surv = 0;
  c->root_slot = root_slot;
  c->pad_slot = pad_slot;
  c->err = 0;
  c->thr_nll = 0.0;
  c->thr_lo = 0ull;
  at<int>(ws, L.r_aux)[0] = 0;
  at<int>(ws, L.b_node)[0] = -1;
  at<double>(ws, L.b_nll)[0] = 0.0;
  at<int>(ws, L.b_depth)[0] = 0;
  at<int>(ws, L.b_lex)[0] = 0;
  at<int>(ws, L.b_slot)[0] = root_slot;
  at<int>(ws, L.b_token)[0] = -1;
  at<int>(ws, L.b_anc)[0] = root_slot;
  at<int>(ws, L.b_anc_len)[0] = 1;
}

// --------------------------------------------------------------------------
// Canonical warp of each batch row (t > 0 scoring): w_rows[b] = apply_warp(row b).
__global__ void __launch_bounds__(kRowThreads) tree_warp_rows_kernel(uint8_t* ws, TreeLayout L, const void* rows,
                                                                       int row_kind, long long ld, double temperature,
                                                                       double top_p, int r0, int r1) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int V = L.V;
  // persistent over the batch rows; the radix-sort scratch belongs to the CTA
  // (kWarpScratchRows rows of V), not to the row -- 148 x V instead of B x V
  const long long sc = (long long)blockIdx.x * V;
  unsigned long long* k1 = at<unsigned long long>(ws, L.w_keys) + sc;
  unsigned long long* k2 = at<unsigned long long>(ws, L.w_keys2) + sc;
  int* i1 = at<int>(ws, L.w_idx) + sc;
  int* i2 = at<int>(ws, L.w_idx2) + sc;
  const int re = rows_end(c, r1);
  for (int b = r0 + blockIdx.x; b < re; b += gridDim.x) {
    const float* z = row_kind == SX_ROWS_LOGITS_F32 ? reinterpret_cast<const float*>(rows) + b * ld : nullptr;
    const double* p = row_kind == SX_ROWS_PROBS_F64 ? reinterpret_cast<const double*>(rows) + b * ld : nullptr;
    double* out = at<double>(ws, L.w_rows) + (long long)b * V;
    warp_row(sm, z, p, V, temperature, top_p, out, k1, i1, k2, i2);
    __syncthreads();  // sm and the scratch are reused by the next row
  }
}

// --------------------------------------------------------------------------
// Row statistics for logits rows: max and canonical sum of exp(z - max).
//
// Threshold prefilter (exact): once the tree holds K candidates, a child can
// only enter if its key beats the threshold, and the threshold only decreases
// (SURVEY Appendix A.7). An fp32 estimate of the child's nll,
//   nll~ = parent_nll - ((z - m) - log S~),  S~ = fp32 sum of __expf(z - m),
// is within 1e-4 of the exact float64 value (|z - m| rounding + S~ relative
// error, both < 2e-5 here), so a candidate with nll~ - kPrefilterSlack >
// thr_nll can never survive: it is dropped without the canonical fp64
// exp/log. A row whose best child (z = m, nll~ = parent_nll + log S~) fails
// that test skips the fp64 sum entirely. Survivors and borderline candidates
// still take the exact path, so the tree is unchanged bit for bit.
constexpr double kPrefilterSlack = 1e-3;

__global__ void __launch_bounds__(kRowThreads) tree_row_stats_kernel(uint8_t* ws, TreeLayout L, const float* rows,
                                                                       long long ld, int r0, int r1) {
  __shared__ RowSmemLite sm;
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int b = r0 + blockIdx.x;
  if (b >= rows_end(c, r1)) return;
  const float* z = rows + b * ld;
  const int V = L.V;
  float mx = -CUDART_INF_F;
  for (int v = threadIdx.x; v < V; v += kRowThreads) mx = fmaxf(mx, z[v]);
  const float m = block_max_f(sm, mx);
  float sa = 0.f;
  for (int v = threadIdx.x; v < V; v += kRowThreads) sa += __expf(z[v] - m);
  for (int o = 16; o > 0; o >>= 1) sa += __shfl_xor_sync(0xffffffff, sa, o);
  if ((threadIdx.x & 31) == 0) sm.redf[threadIdx.x >> 5] = sa;
  __syncthreads();
  float S_est = 0.f;
  for (int w = 0; w < kRowThreads / 32; ++w) S_est += sm.redf[w];
  __syncthreads();
  const float lsa = logf(S_est);
  const double parent_nll = at<double>(ws, L.b_nll)[b];
  const bool skip = c->has_thr && dsub(dadd(parent_nll, (double)lsa), kPrefilterSlack) > c->thr_nll;
  if (skip) {
    if (threadIdx.x == 0) at<float>(ws, L.r_lsa)[b] = -CUDART_INF_F;
    return;
  }
  double acc = 0.0;  // canonical sum (warp_rows.cuh)
  for (int v = threadIdx.x; v < V; v += kRowThreads) acc = dadd(acc, sx_exp(dsub((double)z[v], (double)m)));
  const double S = block_canon_sum(sm, acc);
  if (threadIdx.x == 0) {
    at<float>(ws, L.r_max)[b] = m;
    at<double>(ws, L.r_sum)[b] = S;
    at<float>(ws, L.r_lsa)[b] = lsa;
  }
}

// Argmax rows (t = 0 warped scoring): one child per row with p = 1, edge = log(1) = 0.
__global__ void __launch_bounds__(kRowThreads) tree_argmax_score_kernel(uint8_t* ws, TreeLayout L, const void* rows,
                                                                          int row_kind, long long ld, int r0, int r1) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int b = r0 + blockIdx.x;
  if (b >= rows_end(c, r1)) return;
  double bv = -CUDART_INF;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < L.V; v += kRowThreads) {
    const double x = row_kind == SX_ROWS_LOGITS_F32 ? (double)reinterpret_cast<const float*>(rows)[b * ld + v]
                                                    : reinterpret_cast<const double*>(rows)[b * ld + v];
    if (x > bv) {
      bv = x;
      bi = v;
    }
  }
  const int best = block_argmax(sm, bv, bi);
  if (threadIdx.x == 0) {
    const double parent_nll = at<double>(ws, L.b_nll)[b];
    const double nll = dsub(parent_nll, 0.0);
    const unsigned long long hi = (unsigned long long)__double_as_longlong(nll);
    const unsigned long long lo = make_lo(at<int>(ws, L.b_depth)[b] + 1, at<int>(ws, L.b_lex)[b], best);
    if (!c->has_thr || key_less(hi, lo, (unsigned long long)__double_as_longlong(c->thr_nll), c->thr_lo)) {
      const int k = atomicAdd(&c->n_surv, 1);
      if (k < L.cap) {
        at<double>(ws, L.s_nll)[k] = nll;
        at<unsigned long long>(ws, L.s_lo)[k] = lo;
        at<double>(ws, L.s_edge)[k] = 0.0;
        at<int>(ws, L.s_row)[k] = b;
      } else {
        c->err = 1;
      }
    }
  }
}

// Score every (row, token): grid (chunks, B). mode: probabilities (fp64 rows or the
// warped rows) or logits (fp32 + row stats).
__global__ void __launch_bounds__(256) tree_score_kernel(uint8_t* ws, TreeLayout L, const void* rows, int row_kind,
                                                           long long ld, int r0, int r1) {
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int b = r0 + blockIdx.y;
  if (b >= rows_end(c, r1)) return;
  const int V = L.V;
  const double parent_nll = at<double>(ws, L.b_nll)[b];
  const int depth = at<int>(ws, L.b_depth)[b] + 1;
  const int plex = at<int>(ws, L.b_lex)[b];
  const bool has_thr = c->has_thr;
  const unsigned long long th = (unsigned long long)__double_as_longlong(c->thr_nll);
  const unsigned long long tl = c->thr_lo;
  float m = 0.f;
  double S = 1.0;
  float lsa = 0.f;
  const float* z = nullptr;
  const double* p = nullptr;
  if (row_kind == SX_ROWS_LOGITS_F32) {
    lsa = at<float>(ws, L.r_lsa)[b];
    if (lsa == -CUDART_INF_F) return;  // no child of this row can beat the threshold
    z = reinterpret_cast<const float*>(rows) + b * ld;
    m = at<float>(ws, L.r_max)[b];
    S = at<double>(ws, L.r_sum)[b];
  } else if (row_kind == SX_ROWS_PROBS_F64) {
    p = reinterpret_cast<const double*>(rows) + b * ld;
  } else {
    p = at<double>(ws, L.w_rows) + (long long)b * V;
  }
  const int lane = threadIdx.x & 31;
  for (int v0 = blockIdx.x * blockDim.x; v0 < V; v0 += gridDim.x * blockDim.x) {
    const int v = v0 + threadIdx.x;
    bool keep = false;
    double nll = 0.0, edge = 0.0;
    unsigned long long lo = 0;
    // prefilter (logits rows): drop candidates whose fp32 nll estimate is clearly past the threshold
    const bool pre = v < V && (!z || !has_thr ||
                               !(dsub(dsub(parent_nll, (double)((z[v] - m) - lsa)), kPrefilterSlack) > c->thr_nll));
    if (pre) {
      const double pv = z ? ddiv(sx_exp(dsub((double)z[v], (double)m)), S) : p[v];
      if (pv > 0.0) {
        edge = sx_log(pv);
        nll = dsub(parent_nll, edge);
        lo = make_lo(depth, plex, v);
        keep = !has_thr || key_less((unsigned long long)__double_as_longlong(nll), lo, th, tl);
      }
    }
    const unsigned mask = __ballot_sync(0xffffffff, keep);
    if (mask) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&c->n_surv, __popc(mask));
      base = __shfl_sync(0xffffffff, base, 0);
      if (keep) {
        const long long k = base + __popc(mask & ((1u << lane) - 1));
        if (k < L.cap) {
          at<double>(ws, L.s_nll)[k] = nll;
          at<unsigned long long>(ws, L.s_lo)[k] = lo;
          at<double>(ws, L.s_edge)[k] = edge;
          at<int>(ws, L.s_row)[k] = b;
        } else {
          c->err = 1;
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// Chunked logits-row path (raw scoring of fp32 logits rows), three persistent
// kernels over (row, chunk) work units so that a round of any batch size
// spreads over the whole GPU -- a one-row root round included:
//   max    units of kRowChunkA elements: one HBM read (16-byte streaming loads),
//          chunk max + online fp32 sum of exp(z - max). The last chunk of a row
//          to arrive combines the partials in chunk order: exact row max M and
//          the fp32 estimate S~ (prefilter only). Rows whose best child cannot
//          beat the threshold stop here -- the common case once the tree holds
//          K nodes; the others are appended to the work list.
//   sum    units of kRowChunkB elements of the listed rows: e_v =
//          sx_exp(z_v - M) into the fp64 row scratch; the last chunk to arrive
//          forms the canonical sum (lane t adds e_t, e_t+256, ... then the
//          halving tree -- the order of tree_row_stats_kernel / oxmath.c).
//   score  units of kRowChunkB elements of the listed rows: exact edges
//          sx_log(e_v / S) and keys of the candidates the fp32 estimate cannot
//          rule out; survivors appended.
// Bit-identical to tree_row_stats + tree_score: the prefilter only decides
// which candidates take the exact path (1e-3 of slack against an estimate
// good to ~1e-5), and e_v / S are the same canonical values.
constexpr int kMaxThreads = 128;  // max-pass CTA: small, so >= 1024 of them are resident (one row each at B = 1024)

// kVec: 2 / 3 = pipelined batch-max loop with 4 / 8 x 16 B per thread per batch, 1 = per-element online loop (A/B), 0 = scalar (unaligned rows);
// separate instantiations, so the default path keeps its own (small) register budget
template <int kVec>
__global__ void __launch_bounds__(kMaxThreads) tree_rows_max_kernel(uint8_t* ws, TreeLayout L,
                                                                     const float* __restrict__ rows, long long ld,
                                                                     int r0, int r1) {
  constexpr int vec4 = kVec;
  __shared__ float red_m[kMaxThreads / 32], red_s[kMaxThreads / 32];
  __shared__ int last_s;
  griddep_launch_dependents();  // the sum pass may become resident now (it waits for this grid to finish)
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int batch_n = rows_end(c, r1) - r0, V = L.V, tid = threadIdx.x, lane = tid & 31;
  // Work units: whole rows when the batch fills the grid (no cross-CTA combine),
  // else each row cut into enough chunks (multiples of kRowChunkA elements) to
  // give every CTA work -- the one-row root round spreads over up to 64 CTAs.
  int clen = V;
  if (2 * batch_n <= (int)gridDim.x) {  // whole units per CTA: floor, so no CTA gets one unit more than the rest
    const int per = min(kRowChunksMax, (int)gridDim.x / batch_n);
    clen = ((V + per - 1) / per + kRowChunkA - 1) / kRowChunkA * kRowChunkA;
  }
  const int nch = (V + clen - 1) / clen;
  float* pm = at<float>(ws, L.r_pm);
  float* ps = at<float>(ws, L.r_ps);
  int* cnt = at<int>(ws, L.r_cnt);
  for (int u = blockIdx.x; u < batch_n * nch; u += gridDim.x) {
    const int b = r0 + u / nch, j = u % nch;
    const int v0 = j * clen, v1 = min(V, v0 + clen);
    const float* z = rows + b * ld;
    float m = -CUDART_INF_F, sacc = 0.f;
    auto acc1 = [&](float x) {
      if (x > m) {
        sacc = sacc * __expf(m - x) + 1.f;
        m = x;
      } else {
        sacc += __expf(x - m);
      }
    };
    if constexpr (vec4 >= 2) {
      // chunk bounds are multiples of 4. Register double buffer: the next 4 x 16 B
      // per thread are in flight while the current ones are folded in; per batch
      // one max, one rescale, then independent exps (no per-element branch chain).
      const float4* z4 = reinterpret_cast<const float4*>(z + v0);
      const int n4 = (v1 - v0) >> 2;
      constexpr int U = vec4 == 3 ? 8 : 4;
      const float4 ninf = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
      float4 cur[U], nxt[U];
#pragma unroll
      for (int k = 0; k < U; ++k) cur[k] = tid + k * kMaxThreads < n4 ? __ldcs(z4 + tid + k * kMaxThreads) : ninf;
      float s0 = 0.f, s1 = 0.f;
      for (int i = tid; i < n4; i += U * kMaxThreads) {
        const int in = i + U * kMaxThreads;
#pragma unroll
        for (int k = 0; k < U; ++k) nxt[k] = in + k * kMaxThreads < n4 ? __ldcs(z4 + in + k * kMaxThreads) : ninf;
        float bm = -CUDART_INF_F;
#pragma unroll
        for (int k = 0; k < U; ++k) bm = fmaxf(bm, fmaxf(fmaxf(cur[k].x, cur[k].y), fmaxf(cur[k].z, cur[k].w)));
        if (bm > m) {
          const float r = m == -CUDART_INF_F ? 0.f : __expf(m - bm);
          s0 *= r;
          s1 *= r;
          m = bm;
        }
        if (m != -CUDART_INF_F) {
#pragma unroll
          for (int k = 0; k < U; ++k) {
            s0 += __expf(cur[k].x - m) + __expf(cur[k].y - m);
            s1 += __expf(cur[k].z - m) + __expf(cur[k].w - m);
          }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) cur[k] = nxt[k];
      }
      sacc = s0 + s1;
    } else if constexpr (vec4 == 1) {  // chunk bounds are multiples of 4; 8 loads per thread in flight
      const float4* z4 = reinterpret_cast<const float4*>(z + v0);
      const int n4 = (v1 - v0) >> 2;
      for (int i = tid; i < n4; i += 8 * kMaxThreads) {  // 8 x 16 B per thread in flight, tail included
        float4 a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (i + k * kMaxThreads < n4) a[k] = __ldcs(z4 + i + k * kMaxThreads);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (i + k * kMaxThreads < n4) acc1(a[k].x), acc1(a[k].y), acc1(a[k].z), acc1(a[k].w);
      }
    } else {
      for (int v = v0 + tid; v < v1; v += kMaxThreads) acc1(z[v]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sacc, o);
      const float mm = fmaxf(m, m2);
      sacc = (m == -CUDART_INF_F ? 0.f : sacc * __expf(m - mm)) + (m2 == -CUDART_INF_F ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      red_m[tid >> 5] = m;
      red_s[tid >> 5] = sacc;
    }
    __syncthreads();
    if (tid == 0) {
      float M = red_m[0];
      for (int w = 1; w < kMaxThreads / 32; ++w) M = fmaxf(M, red_m[w]);
      float S = 0.f;
      for (int w = 0; w < kMaxThreads / 32; ++w)
        if (red_m[w] != -CUDART_INF_F) S += red_s[w] * __expf(red_m[w] - M);
      if (nch > 1) {
        pm[b * kRowChunksMax + j] = M;
        ps[b * kRowChunksMax + j] = S;
        __threadfence();
        last_s = atomicAdd(&cnt[b], 1) == nch - 1;
      } else {
        last_s = 1;
        red_m[0] = M;
        red_s[0] = S;
      }
    }
    __syncthreads();
    if (last_s && tid < 32) {  // warp 0 finishes the row (the last of its chunks to arrive)
      float RM = red_m[0], RS = red_s[0];
      if (nch > 1) {  // combine the partials (nch <= 64: two per lane, fixed shuffle order)
        __threadfence();
        const float m0 = lane < nch ? __ldcg(pm + b * kRowChunksMax + lane) : -CUDART_INF_F;
        const float m1 = lane + 32 < nch ? __ldcg(pm + b * kRowChunksMax + lane + 32) : -CUDART_INF_F;
        const float s0 = lane < nch ? __ldcg(ps + b * kRowChunksMax + lane) : 0.f;
        const float s1 = lane + 32 < nch ? __ldcg(ps + b * kRowChunksMax + lane + 32) : 0.f;
        RM = fmaxf(m0, m1);
        for (int o = 16; o > 0; o >>= 1) RM = fmaxf(RM, __shfl_xor_sync(0xffffffffu, RM, o));
        RS = (m0 == -CUDART_INF_F ? 0.f : s0 * __expf(m0 - RM)) + (m1 == -CUDART_INF_F ? 0.f : s1 * __expf(m1 - RM));
        for (int o = 16; o > 0; o >>= 1) RS += __shfl_xor_sync(0xffffffffu, RS, o);
      }
      if (lane == 0) {
        const float lsa = logf(RS);
        const double parent_nll = at<double>(ws, L.b_nll)[b];
        const bool skip = c->has_thr && dsub(dadd(parent_nll, (double)lsa), kPrefilterSlack) > c->thr_nll;
        at<float>(ws, L.r_max)[b] = RM;
        at<float>(ws, L.r_lsa)[b] = skip ? -CUDART_INF_F : lsa;
        if (nch > 1) cnt[b] = 0;
        if (!skip) at<int>(ws, L.r_list)[atomicAdd(at<int>(ws, L.r_aux), 1)] = b;
      }
    }
    __syncthreads();  // red_* reused by the next unit
  }
}

// One sum unit (row r_list[w], chunk j): e_v = exp(z_v - M) into the fp64 row
// scratch; the last chunk to arrive forms the canonical row sum. `ready` != null
// (fused exact pass): the sum's writer then publishes ready[b] = stamp.
SX_DEV void rows_sum_unit(uint8_t* ws, const TreeLayout& L, const float* __restrict__ rows, long long ld, int u,
                          int nch, RowSmemLite& sm, int& last, int* ready, int stamp) {
  const int V = L.V, tid = threadIdx.x;
  int* cnt = at<int>(ws, L.r_cnt) + L.B;
  const int w = u / nch, j = u - w * nch;
  const int b = at<int>(ws, L.r_list)[w];
  const float* z = rows + b * ld;
  const double M = (double)at<float>(ws, L.r_max)[b];
  double* e = at<double>(ws, L.w_rows) + (long long)b * V;
  const int v1 = min(V, (j + 1) * kRowChunkB);
  for (int v = j * kRowChunkB + tid; v < v1; v += kRowThreads) e[v] = sx_exp(dsub((double)z[v], M));
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(&cnt[b], 1) == nch - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    double acc = 0.0;  // canonical sum: lane t adds e_t, e_t+256, ... in order
    int v = tid;
    for (; v + 7 * kRowThreads < V; v += 8 * kRowThreads) {  // 8 independent loads, then the ordered adds
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = __ldcg(e + v + k * kRowThreads);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = dadd(acc, x[k]);
    }
    for (; v < V; v += kRowThreads) acc = dadd(acc, __ldcg(e + v));
    const double S = block_canon_sum(sm, acc);
    if (tid == 0) {
      at<double>(ws, L.r_sum)[b] = S;
      cnt[b] = 0;
      if (ready) {
        __threadfence();
        atomicExch(&ready[b], stamp);
      }
    }
  }
}

// One score unit: exact edges log(e_v / S) and keys of the candidates the fp32
// estimate cannot rule out; survivors appended. kFused: the row's e_v and S were
// written by other CTAs of this grid, so they are read through L2 (__ldcg).
template <bool kFused>
SX_DEV void rows_score_unit(uint8_t* ws, const TreeLayout& L, const float* __restrict__ rows, long long ld, int u,
                            int nch) {
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int V = L.V, tid = threadIdx.x, lane = tid & 31;
  const bool has_thr = c->has_thr;
  const double thr_nll = c->thr_nll;
  const unsigned long long th = (unsigned long long)__double_as_longlong(thr_nll);
  const unsigned long long tl = c->thr_lo;
  const int w = u / nch, j = u - w * nch;
  const int b = at<int>(ws, L.r_list)[w];
  const float* z = rows + b * ld;
  const float M = at<float>(ws, L.r_max)[b], lsa = at<float>(ws, L.r_lsa)[b];
  const double S = kFused ? __ldcg(at<double>(ws, L.r_sum) + b) : at<double>(ws, L.r_sum)[b];
  const double parent_nll = at<double>(ws, L.b_nll)[b];
  const int depth = at<int>(ws, L.b_depth)[b] + 1;
  const int plex = at<int>(ws, L.b_lex)[b];
  const double* e = at<double>(ws, L.w_rows) + (long long)b * V;
  const int v0 = j * kRowChunkB;
  for (int vb = v0; vb < v0 + kRowChunkB; vb += kRowThreads) {  // whole warps iterate (ballot)
    const int v = vb + tid;
    bool keep = false;
    double nll = 0.0, edge = 0.0;
    unsigned long long lo = 0;
    if (v < V) {
      const float zv = z[v];
      if (!has_thr || !(dsub(dsub(parent_nll, (double)((zv - M) - lsa)), kPrefilterSlack) > thr_nll)) {
        const double pv = ddiv(kFused ? __ldcg(e + v) : e[v], S);
        if (pv > 0.0) {
          edge = sx_log(pv);
          nll = dsub(parent_nll, edge);
          lo = make_lo(depth, plex, v);
          keep = !has_thr || key_less((unsigned long long)__double_as_longlong(nll), lo, th, tl);
        }
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&c->n_surv, __popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep) {
        const long long k = base + __popc(mask & ((1u << lane) - 1));
        if (k < L.cap) {
          at<double>(ws, L.s_nll)[k] = nll;
          at<unsigned long long>(ws, L.s_lo)[k] = lo;
          at<double>(ws, L.s_edge)[k] = edge;
          at<int>(ws, L.s_row)[k] = b;
        } else {
          c->err = 1;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kRowThreads) tree_rows_sum_kernel(uint8_t* ws, TreeLayout L,
                                                                     const float* __restrict__ rows, long long ld) {
  __shared__ RowSmemLite sm;
  __shared__ int last;
  griddep_wait();  // launched early (programmatic stream serialization): the max pass's work list
  griddep_launch_dependents();
  const int nwork = *(volatile int*)at<int>(ws, L.r_aux);
  const int nch = (L.V + kRowChunkB - 1) / kRowChunkB;
  for (int u = blockIdx.x; u < nwork * nch; u += gridDim.x) rows_sum_unit(ws, L, rows, ld, u, nch, sm, last, nullptr, 0);
}

__global__ void __launch_bounds__(kRowThreads) tree_rows_score_kernel(uint8_t* ws, TreeLayout L,
                                                                       const float* __restrict__ rows, long long ld) {
  griddep_wait();  // launched early: the sums of the listed rows
  griddep_launch_dependents();
  const int nwork = at<int>(ws, L.r_aux)[0];
  const int nch = (L.V + kRowChunkB - 1) / kRowChunkB;
  for (int u = blockIdx.x; u < nwork * nch; u += gridDim.x) rows_score_unit<false>(ws, L, rows, ld, u, nch);
}

// Fused exact pass (the default): the sum and score units of the listed rows in
// ONE persistent grid (<= the resident CTAs, so every CTA is resident): each CTA
// first takes its sum units, then its score units, and a score unit waits for
// its row's readiness flag (ready[b] == this round's stamp, r_aux[1] + 1; the
// update kernel advances r_aux[1] every round, so stale flags never match) --
// one kernel boundary less per round, and with an empty work list one launch
// instead of two. The successor (the update) is released only at the end:
// it must not take SM resources a not-yet-resident CTA of this grid needs.
__global__ void __launch_bounds__(kRowThreads) tree_rows_exact_kernel(uint8_t* ws, TreeLayout L,
                                                                       const float* __restrict__ rows, long long ld) {
  __shared__ RowSmemLite sm;
  __shared__ int last;
  griddep_wait();  // launched early: the max pass's work list
  const int nwork = *(volatile int*)at<int>(ws, L.r_aux);
  const int stamp = *(volatile int*)(at<int>(ws, L.r_aux) + 1) + 1;
  int* ready = at<int>(ws, L.r_ready);
  const int nch = (L.V + kRowChunkB - 1) / kRowChunkB;
  const int units = nwork * nch;
  for (int u = blockIdx.x; u < units; u += gridDim.x) rows_sum_unit(ws, L, rows, ld, u, nch, sm, last, ready, stamp);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = at<int>(ws, L.r_list)[u / nch];
    if (threadIdx.x == 0)
      while (*(volatile int*)(ready + b) != stamp) __nanosleep(64);
    __syncthreads();
    __threadfence();
    rows_score_unit<true>(ws, L, rows, ld, u, nch);
  }
  griddep_launch_dependents();
}

// --------------------------------------------------------------------------
// The single-CTA update: select, sort, relabel, threshold, next batch.
constexpr int kUpdThreads = 1024;
constexpr int kUpdCluster = 8;  // CTAs sharing the radix-select histograms (portable cluster size)
constexpr int kUpdBatch = 8;    // independent key loads per thread before the histogram votes

struct UpdSmem {
  int hist[2][256];  // this CTA's histogram of the current digit (double-buffered across digits)
  int wsum[8];
  int bin;
  int rank;
  int done;
  int sel_n;
  int elig_total;
  int scan[kUpdThreads];
  int depth_start[256];
  int wscan[kUpdThreads / 32 + 1];  // block_excl_scan_fast: per-warp totals, exclusive-scanned
};

SX_DEV void get_key(uint8_t* ws, const TreeLayout& L, int cur, int n_old, int i, unsigned long long& h,
                    unsigned long long& l) {
  if (i < n_old) {
    h = (unsigned long long)__double_as_longlong(at<double>(ws, L.m_nll[cur])[i]);
    l = at<unsigned long long>(ws, L.m_lo[cur])[i];
  } else {
    h = (unsigned long long)__double_as_longlong(at<double>(ws, L.s_nll)[i - n_old]);
    l = at<unsigned long long>(ws, L.s_lo)[i - n_old];
  }
}

SX_DEV int digit_of(unsigned long long h, unsigned long long l, int d) {
  return d < 8 ? (int)((h >> (56 - 8 * d)) & 255) : (int)((l >> (56 - 8 * (d - 8))) & 255);
}
// compare top (d+1) digits of key against prefix digits: -1, 0, +1
SX_DEV int cmp_prefix(unsigned long long h, unsigned long long l, unsigned long long ph, unsigned long long pl,
                      int ndig) {
  if (ndig <= 8) {
    const int sh = 64 - 8 * ndig;
    const unsigned long long a = sh >= 64 ? 0 : (h >> sh), b = sh >= 64 ? 0 : (ph >> sh);
    return a < b ? -1 : (a > b ? 1 : 0);
  }
  if (h != ph) return h < ph ? -1 : 1;
  const int sh = 64 - 8 * (ndig - 8);
  const unsigned long long a = sh >= 64 ? 0 : (l >> sh), b = sh >= 64 ? 0 : (pl >> sh);
  return a < b ? -1 : (a > b ? 1 : 0);
}

SX_DEV void bitonic_sort_128(unsigned long long* kh, unsigned long long* kl, int* kv, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool asc = (i & k) == 0;
          const bool gt = key_less(kh[ixj], kl[ixj], kh[i], kl[i]);
          if (gt == asc) {
            unsigned long long th = kh[i], tl = kl[i];
            int tv = kv[i];
            kh[i] = kh[ixj];
            kl[i] = kl[ixj];
            kv[i] = kv[ixj];
            kh[ixj] = th;
            kl[ixj] = tl;
            kv[ixj] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

SX_DEV void bitonic_sort_64(unsigned long long* kk, int* kv, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool asc = (i & k) == 0;
          if ((kk[i] > kk[ixj]) == asc) {
            unsigned long long t = kk[i];
            int tv = kv[i];
            kk[i] = kk[ixj];
            kv[i] = kv[ixj];
            kk[ixj] = t;
            kv[ixj] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Register-resident bitonic sort of n = 2^m (64 <= n <= 8 * kUpdThreads) keys
// held in shared memory (kh:kl 128-bit, or kl alone when !kWide; values kv),
// ascending, identical result to bitonic_sort_128 / bitonic_sort_64 (the same
// compare-exchange network). Thread t of T = min(n, blockDim.x) holds elements
// i = e*T + t, e < n / T: partner distance j < 32 -> warp shuffle, j >= T ->
// the thread's own registers, otherwise one shared-memory exchange (2 barriers).
// n = 1024: 40 of the 55 stages stay in registers.
// make TRACE=1: the update kernel's CTA 0 stamps %globaltimer at its phase
// boundaries into r_aux[16..48) (8-byte slots; tools/tree_round_bench.py --trace)
#ifdef SX_TREE_TRACE
SX_DEV void trace_mark(uint8_t* ws, const TreeLayout& L, int slot) {
  if (threadIdx.x == 0 && cluster_ctarank() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    reinterpret_cast<unsigned long long*>(at<int>(ws, L.r_aux) + 16)[slot] = t;
  }
}
#define SX_TRACE(slot) trace_mark(ws, L, slot)
#else
#define SX_TRACE(slot) ((void)0)
#endif

// SX_TREE_SORT_REG=0: the shared-memory network for every stage (A/B)
__constant__ int g_sort_reg = 1;
// SX_TREE_MERGE=0: radix select + sort of the union in every round (A/B)
__constant__ int g_update_merge = 1;

template <bool kWide, int EM>
SX_DEV void bitonic_sort_reg_e(unsigned long long* kh, unsigned long long* kl, int* kv, int n) {
  const int T = n < (int)blockDim.x ? n : (int)blockDim.x;
  const int E = n / T;
  const int t = threadIdx.x;
  const bool act = t < T;
  unsigned long long h[EM], l[EM];
  int v[EM];
#pragma unroll
  for (int e = 0; e < EM; ++e) {
    h[e] = l[e] = 0;
    v[e] = 0;
    if (act && e < E) {
      const int i = e * T + t;
      if (kWide) h[e] = kh[i];
      l[e] = kl[i];
      v[e] = kv[i];
    }
  }
  auto less = [&](unsigned long long ah, unsigned long long al, unsigned long long bh, unsigned long long bl) {
    return kWide ? (ah < bh || (ah == bh && al < bl)) : (al < bl);
  };
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= T) {  // partner in this thread: slot e ^ (j / T) (compile-time slots: no local-memory arrays)
        const int js = j / T;
#pragma unroll
        for (int e = 0; e < EM; ++e) {
#pragma unroll
          for (int pe = e + 1; pe < EM; ++pe) {
            if ((e ^ pe) == js && act) {
              const int i = e * T + t;
              const bool asc = (i & k) == 0;
              if (less(h[pe], l[pe], h[e], l[e]) == asc) {
                const unsigned long long th = h[e], tl = l[e];
                const int tv = v[e];
                h[e] = h[pe], l[e] = l[pe], v[e] = v[pe];
                h[pe] = th, l[pe] = tl, v[pe] = tv;
              }
            }
          }
        }
      } else if (j < 32) {  // partner lane t ^ j, same slot
#pragma unroll
        for (int e = 0; e < EM; ++e) {
          if (e < E) {
            const int i = e * T + t;
            const unsigned long long ph = kWide ? __shfl_xor_sync(0xffffffffu, h[e], j) : 0ull;
            const unsigned long long pl = __shfl_xor_sync(0xffffffffu, l[e], j);
            const int pv = __shfl_xor_sync(0xffffffffu, v[e], j);
            // the compare-exchange of bitonic_sort_128: swap iff (upper < lower) == asc
            const bool asc = (i & k) == 0;
            const bool swap = ((i & j) == 0) ? (less(ph, pl, h[e], l[e]) == asc) : (less(h[e], l[e], ph, pl) == asc);
            if (swap) h[e] = ph, l[e] = pl, v[e] = pv;
          }
        }
      } else {  // partner thread t ^ j: exchange through shared memory
#pragma unroll
        for (int e = 0; e < EM; ++e)
          if (act && e < E) {
            const int i = e * T + t;
            if (kWide) kh[i] = h[e];
            kl[i] = l[e];
            kv[i] = v[e];
          }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EM; ++e) {
          if (act && e < E) {
            const int i = e * T + t, p = i ^ j;
            const unsigned long long ph = kWide ? kh[p] : 0ull, pl = kl[p];
            const bool asc = (i & k) == 0;
            const bool swap = ((i & j) == 0) ? (less(ph, pl, h[e], l[e]) == asc) : (less(h[e], l[e], ph, pl) == asc);
            if (swap) h[e] = ph, l[e] = pl, v[e] = kv[p];
          }
        }
        __syncthreads();
      }
    }
  }
#pragma unroll
  for (int e = 0; e < EM; ++e)
    if (act && e < E) {
      const int i = e * T + t;
      if (kWide) kh[i] = h[e];
      kl[i] = l[e];
      kv[i] = v[e];
    }
  __syncthreads();
}

template <bool kWide>
SX_DEV void bitonic_sort_reg(unsigned long long* kh, unsigned long long* kl, int* kv, int n) {
  const int E = n / (int)blockDim.x;
  if (E <= 1)
    bitonic_sort_reg_e<kWide, 1>(kh, kl, kv, n);
  else if (E == 2)
    bitonic_sort_reg_e<kWide, 2>(kh, kl, kv, n);
  else if (E == 4)
    bitonic_sort_reg_e<kWide, 4>(kh, kl, kv, n);
  else
    bitonic_sort_reg_e<kWide, 8>(kh, kl, kv, n);
}

// block-wide exclusive scan of one int per thread (warp shuffles + one pass over
// the 32 warp totals: 2 barriers); returns the total
SX_DEV int block_excl_scan_fast(UpdSmem& sm, int v, int& excl) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.wscan[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = kUpdThreads / 32;
    const int t = lane < nw ? sm.wscan[lane] : 0;
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sm.wscan[lane] = s - t;
    if (lane == 31) sm.wscan[nw] = s;
  }
  __syncthreads();
  excl = sm.wscan[w] + x - v;
  const int total = sm.wscan[kUpdThreads / 32];
  __syncthreads();  // wscan is reused by the next call
  return total;
}

// block-wide exclusive scan of one int per thread; returns the total
SX_DEV int block_excl_scan(UpdSmem& sm, int v, int& excl) {
  const int t = threadIdx.x;
  sm.scan[t] = v;
  __syncthreads();
  for (int off = 1; off < kUpdThreads; off <<= 1) {
    const int add = t >= off ? sm.scan[t - off] : 0;
    __syncthreads();
    sm.scan[t] += add;
    __syncthreads();
  }
  const int incl = sm.scan[t];
  const int total = sm.scan[kUpdThreads - 1];
  __syncthreads();
  excl = incl - v;
  return total;
}

// final = 0: merge only (a slice of an overflowed round, sx_tree_round_rows): the
// materialized list, lex ranks and threshold take in this slice's survivors and
// the current batch is remapped to the new positions; the next batch is picked
// by the last slice (final = 1), as in an ordinary round.
__global__ void __launch_bounds__(kUpdThreads, 1) tree_update_kernel(uint8_t* ws, TreeLayout L, int final) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  UpdSmem& sm = *reinterpret_cast<UpdSmem*>(smem_raw);
  unsigned long long* sk_h = reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(UpdSmem) + 15) & ~size_t(15)));
  unsigned long long* sk_l = sk_h + L.kpad;
  int* sk_v = reinterpret_cast<int*>(sk_l + L.kpad);

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned crank = cluster.block_rank();
  SX_TRACE(0);
  griddep_wait();  // launched early (chunked row path): the survivors of this round
  SX_TRACE(1);
  if (crank == 0 && threadIdx.x == 0) ++at<int>(ws, L.r_aux)[1];  // round stamp of the fused exact pass
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int tid = threadIdx.x;
  const int K = L.K;
  if (c->err) {
    // survivor buffer overflow: some candidates of this round were dropped, so
    // leave the tree untouched; the host re-runs the round in row slices whose
    // survivors fit (sx_tree_round_rows). err stays set for the host to see.
    if (crank == 0 && tid == 0) {
      c->n_surv = 0;
      at<int>(ws, L.r_aux)[0] = 0;
    }
    return;
  }
  const int cur = c->cur, nxt = cur ^ 1;
  const int n_old = c->count;
  const int n_new = min((long long)c->n_surv, L.cap);
  const int n = n_old + n_new;
  // every CTA has read the control block before CTA 0 can rewrite it: CTA 0 only
  // writes after the cluster barriers of steps 1-2 (n_new > 0), and with
  // n_new == 0 the other CTAs have nothing to do
  if (n_new == 0 && crank != 0) return;
  // Merge path: the materialized list is already sorted by key (relabelling lex
  // ranks is monotone within a depth, so it stays sorted across rounds), so when
  // the survivors fit the sort buffer, CTA 0 sorts just them and merges the two
  // runs -- the same K smallest keys in the same order as select + sort of the union
  const bool merge_path = g_update_merge && n_old > 0 && n_new <= L.kpad && L.kpad >= 64;
  if (merge_path && crank != 0) return;
  const int i0 = (int)((long long)n * crank / kUpdCluster), i1 = (int)((long long)n * (crank + 1) / kUpdCluster);
  int* lex;
  const int* par;
  unsigned long long* lo_arr;
  int sel, dst;
  bool has_thr;
  unsigned long long th, tl;
  if (n_new == 0 && !final) {  // merge-only slice with nothing to merge
    if (tid == 0) at<int>(ws, L.r_aux)[0] = 0;
    return;
  }
  if (n_new == 0) {
    // no candidate beat the threshold (every row prefiltered away, or only
    // zero-probability tokens): the materialized list, its lex ranks and the
    // threshold are unchanged -- only the next batch is picked (steps 1-5 would
    // reproduce the same sorted list bit for bit)
    dst = cur;
    sel = n_old;
    lex = at<int>(ws, L.m_lex[cur]);
    par = at<int>(ws, L.m_parent[cur]);
    lo_arr = at<unsigned long long>(ws, L.m_lo[cur]);
    has_thr = c->has_thr;
    th = (unsigned long long)__double_as_longlong(c->thr_nll);
    tl = c->thr_lo;
  } else {
    dst = nxt;

  int np2 = 1;  // power of two >= sel (the lex sort below)
  if (merge_path) {
    sel = min(n, K);
    while (np2 < sel) np2 <<= 1;
    // survivors -> shared memory, sorted (register bitonic network; pads sort last)
    int np2s = 64;
    while (np2s < n_new) np2s <<= 1;
    for (int j = tid; j < np2s; j += kUpdThreads) {
      if (j < n_new) {
        sk_h[j] = (unsigned long long)__double_as_longlong(at<double>(ws, L.s_nll)[j]);
        sk_l[j] = at<unsigned long long>(ws, L.s_lo)[j];
        sk_v[j] = n_old + j;
      } else {
        sk_h[j] = ~0ull;
        sk_l[j] = ~0ull;
        sk_v[j] = -1;
      }
    }
    __syncthreads();
    bitonic_sort_reg<true>(sk_h, sk_l, sk_v, np2s);
    // merge path over the output positions [0, sel): thread t takes [o0, o1); the
    // split (i old, o - i survivors) is the merge-path diagonal (keys are unique)
    const double* a_nll = at<double>(ws, L.m_nll[cur]);
    const unsigned long long* a_lo = at<unsigned long long>(ws, L.m_lo[cur]);
    constexpr int kMergeMax = 8;  // sel <= 8192 = 8 x kUpdThreads
    const int per_o = (sel + kUpdThreads - 1) / kUpdThreads;
    const int o0 = min(sel, tid * per_o), o1 = min(sel, o0 + per_o);
    unsigned long long oh[kMergeMax], ol[kMergeMax];
    int ov[kMergeMax];
    {
      // smallest i in [max(0, o0 - n_new), min(o0, n_old)] with A[i] > S[o0 - i - 1]
      int lo_i = max(0, o0 - n_new), hi_i = min(o0, n_old);
      while (lo_i < hi_i) {
        const int mid = (lo_i + hi_i) >> 1;
        const int j = o0 - mid - 1;  // compare A[mid] with S[j]
        const unsigned long long ah = (unsigned long long)__double_as_longlong(a_nll[mid]);
        if (key_less(sk_h[j], sk_l[j], ah, a_lo[mid]))
          hi_i = mid;  // S[j] < A[mid]: A[mid] comes after S[j], so fewer than mid+1 old before o0
        else
          lo_i = mid + 1;
      }
      int i = lo_i, j = o0 - lo_i;
      unsigned long long ah = i < n_old ? (unsigned long long)__double_as_longlong(a_nll[i]) : ~0ull;
      unsigned long long al = i < n_old ? a_lo[i] : ~0ull;
#pragma unroll
      for (int k = 0; k < kMergeMax; ++k) {
        if (o0 + k < o1) {
          const bool take_s = j < n_new && (i >= n_old || key_less(sk_h[j], sk_l[j], ah, al));
          if (take_s) {
            oh[k] = sk_h[j];
            ol[k] = sk_l[j];
            ov[k] = sk_v[j];
            ++j;
          } else {
            oh[k] = ah;
            ol[k] = al;
            ov[k] = i;
            ++i;
            ah = i < n_old ? (unsigned long long)__double_as_longlong(a_nll[i]) : ~0ull;
            al = i < n_old ? a_lo[i] : ~0ull;
          }
        }
      }
    }
    __syncthreads();  // every thread has read the survivor run
#pragma unroll
    for (int k = 0; k < kMergeMax; ++k)
      if (o0 + k < o1) {
        sk_h[o0 + k] = oh[k];
        sk_l[o0 + k] = ol[k];
        sk_v[o0 + k] = ov[k];
      }
    __syncthreads();
  } else {
  // ---- 1. select the K smallest keys (radix select over 16 8-bit digits) ----
  // Every CTA of the cluster histograms its slice [i0, i1) of the n keys; the
  // 256-bin totals are summed over DSMEM and scanned in parallel by every CTA.
  unsigned long long ph = 0, pl = 0;
  int ndig = 0;  // digits fixed in the prefix
  const bool select_all = n <= K;
  if (!select_all) {
    int rank = K;
    for (int d = 0; d < 16; ++d) {
      int* h = sm.hist[d & 1];
      if (tid < 256) h[tid] = 0;
      __syncthreads();
      // kUpdBatch independent key loads per thread, then the votes (uniform trip count)
      for (int base = i0; base < i1; base += kUpdThreads * kUpdBatch) {
        unsigned long long kh[kUpdBatch], kl[kUpdBatch];
#pragma unroll
        for (int r = 0; r < kUpdBatch; ++r) {
          const int i = base + r * kUpdThreads + tid;
          kh[r] = kl[r] = 0;
          if (i < i1) {
            if (d < 8)  // digits 0..7 and their prefix need only the nll bits
              kh[r] = (unsigned long long)__double_as_longlong(i < n_old ? at<double>(ws, L.m_nll[cur])[i]
                                                                        : at<double>(ws, L.s_nll)[i - n_old]);
            else
              get_key(ws, L, cur, n_old, i, kh[r], kl[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < kUpdBatch; ++r) {
          const int i = base + r * kUpdThreads + tid;
          const int dig = (i < i1 && cmp_prefix(kh[r], kl[r], ph, pl, d) == 0) ? digit_of(kh[r], kl[r], d) : -1;
          // warp-aggregated increments: the leading digits are shared by most keys,
          // so per-key shared atomics would serialise on one bin
          const unsigned same = __match_any_sync(0xffffffffu, dig);
          if (dig >= 0 && (tid & 31) == __ffs(same) - 1) atomicAdd(&h[dig], __popc(same));
        }
      }
      // the peers' histograms of digit d are complete (and every peer has finished
      // reading digit d-1's buffer, which digit d+1 zeroes)
      cluster.sync();
      int v = 0, x = 0;
      if (tid < 256) {
        for (int r = 0; r < kUpdCluster; ++r) v += cluster.map_shared_rank(h, r)[tid];
        x = v;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if ((tid & 31) >= o) x += y;
        }
        if ((tid & 31) == 31) sm.wsum[tid >> 5] = x;
      }
      __syncthreads();
      if (tid < 256) {
        for (int w = 0; w < (tid >> 5); ++w) x += sm.wsum[w];
        const int excl = x - v;
        if (excl < rank && rank <= x) {  // the bin holding the rank-th smallest key
          sm.bin = tid;
          sm.rank = rank - excl;
          sm.done = (v == rank - excl);
        }
      }
      __syncthreads();
      const unsigned long long bd = (unsigned long long)sm.bin;
      if (d < 8)
        ph |= bd << (56 - 8 * d);
      else
        pl |= bd << (56 - 8 * (d - 8));
      ndig = d + 1;
      rank = sm.rank;
      const int done = sm.done;
      __syncthreads();
      if (done) break;
    }
  }

  // ---- 2. gather the selected keys into CTA 0's shared memory ----
  if (tid == 0) sm.sel_n = 0;
  __syncthreads();
  for (int base = i0; base < i1; base += kUpdThreads * kUpdBatch) {
    unsigned long long h[kUpdBatch], l[kUpdBatch];
#pragma unroll
    for (int r = 0; r < kUpdBatch; ++r) {
      const int i = base + r * kUpdThreads + tid;
      if (i < i1) get_key(ws, L, cur, n_old, i, h[r], l[r]);
    }
#pragma unroll
    for (int r = 0; r < kUpdBatch; ++r) {
      const int i = base + r * kUpdThreads + tid;
      if (i < i1 && (select_all || cmp_prefix(h[r], l[r], ph, pl, ndig) <= 0)) {
        const int k = atomicAdd(&sm.sel_n, 1);
        sk_h[k] = h[r];
        sk_l[k] = l[r];
        sk_v[k] = i;
      }
    }
  }
  cluster.sync();  // every CTA's local count is final
  if (crank != 0) {  // append this CTA's keys after those of lower ranks, in CTA 0
    int base = 0;
    for (unsigned r = 0; r < crank; ++r) base += *cluster.map_shared_rank(&sm.sel_n, r);
    unsigned long long* dh = cluster.map_shared_rank(sk_h, 0u);
    unsigned long long* dl = cluster.map_shared_rank(sk_l, 0u);
    int* dv = cluster.map_shared_rank(sk_v, 0u);
    for (int k = tid; k < sm.sel_n; k += kUpdThreads) {
      dh[base + k] = sk_h[k];
      dl[base + k] = sk_l[k];
      dv[base + k] = sk_v[k];
    }
  } else if (tid == 0) {
    int tot = 0;
    for (int r = 0; r < kUpdCluster; ++r) tot += *cluster.map_shared_rank(&sm.sel_n, r);
    sm.elig_total = tot;
  }
  cluster.sync();  // CTA 0 holds every selected key; nobody touches a peer's smem after this
  if (crank != 0) return;
  sel = sm.elig_total;  // == min(n, K)
  while (np2 < sel) np2 <<= 1;
  for (int i = sel + tid; i < np2; i += kUpdThreads) {
    sk_h[i] = ~0ull;
    sk_l[i] = ~0ull;
    sk_v[i] = -1;
  }
  __syncthreads();
  if (np2 >= 64 && g_sort_reg)
    bitonic_sort_reg<true>(sk_h, sk_l, sk_v, np2);
  else
    bitonic_sort_128(sk_h, sk_l, sk_v, np2);
  }  // select + sort

  SX_TRACE(2);
  // ---- 3. write the new materialized list (sorted), remap old -> new ----
  int* remap = at<int>(ws, L.remap);
  int* b_node = at<int>(ws, L.b_node);
  for (int i = tid; i < n_old; i += kUpdThreads) remap[i] = -1;  // pruned unless selected
  __syncthreads();
  for (int pos = tid; pos < sel; pos += kUpdThreads) {
    const int src = sk_v[pos];
    if (src < n_old) remap[src] = pos;
  }
  __syncthreads();
  for (int pos = tid; pos < sel; pos += kUpdThreads) {
    const int src = sk_v[pos];
    int parent_old, slot;
    double edge;
    if (src < n_old) {
      parent_old = at<int>(ws, L.m_parent[cur])[src];
      slot = at<int>(ws, L.m_slot[cur])[src];
      edge = at<double>(ws, L.m_edge[cur])[src];
    } else {
      const int j = src - n_old;
      parent_old = b_node[at<int>(ws, L.s_row)[j]];
      slot = -1;
      edge = at<double>(ws, L.s_edge)[j];
    }
    at<double>(ws, L.m_nll[nxt])[pos] = __longlong_as_double((long long)sk_h[pos]);
    at<unsigned long long>(ws, L.m_lo[nxt])[pos] = sk_l[pos];
    at<double>(ws, L.m_edge[nxt])[pos] = edge;
    at<int>(ws, L.m_parent[nxt])[pos] = parent_old < 0 ? -1 : remap[parent_old];
    at<int>(ws, L.m_slot[nxt])[pos] = slot;
  }
  __syncthreads();

  SX_TRACE(3);
  // ---- 4. lex ranks within depth: order by the lo keys (depth | lex(parent) | token) ----
  lex = at<int>(ws, L.m_lex[nxt]);
  const unsigned long long* lo_new = at<unsigned long long>(ws, L.m_lo[nxt]);
  if (merge_path) {
    // The kept old nodes are already in lex order (their old lex ranks; removing
    // nodes or relabelling parents preserves it), so only the new nodes are
    // sorted, then the two runs are merged -- the order the full sort gives.
    const unsigned long long* lo_old = at<unsigned long long>(ws, L.m_lo[cur]);
    const int* lex_old = at<int>(ws, L.m_lex[cur]);
    int* ds_old = sm.hist[0];  // exclusive depth starts of the old list (the histograms are unused here)
    int* ds_new = sm.hist[1];  // ... and of the new list (= sm.depth_start of the sort path)
    for (int i = tid; i < 256; i += kUpdThreads) ds_old[i] = ds_new[i] = 0;
    __syncthreads();
    for (int pos = tid; pos < n_old; pos += kUpdThreads) atomicAdd(&ds_old[lo_depth(lo_old[pos])], 1);
    for (int pos = tid; pos < sel; pos += kUpdThreads) atomicAdd(&ds_new[lo_depth(lo_new[pos])], 1);
    __syncthreads();
    if (tid == 0 || tid == 32) {
      int* a = tid == 0 ? ds_old : ds_new;
      int s = 0;
      for (int i = 0; i < 256; ++i) {
        const int c = a[i];
        a[i] = s;
        s += c;
      }
    }
    int* a_raw = reinterpret_cast<int*>(sk_h);  // [kpad]: old list in lex order -> new position or -1
    int* mark = a_raw + L.kpad;                  // [kpad]: 1 = new node
    for (int pos = tid; pos < sel; pos += kUpdThreads) mark[pos] = 1;
    if (tid == 0) sm.sel_n = 0;
    __syncthreads();
    for (int pos = tid; pos < n_old; pos += kUpdThreads) {
      const int r = remap[pos];
      a_raw[ds_old[lo_depth(lo_old[pos])] + lex_old[pos]] = r;
      if (r >= 0) mark[r] = 0;
    }
    __syncthreads();
    for (int pos = tid; pos < sel; pos += kUpdThreads)
      if (mark[pos]) {
        const int k = atomicAdd(&sm.sel_n, 1);
        sk_l[k] = lo_new[pos];
        sk_v[k] = pos;
      }
    __syncthreads();
    const int nb = sm.sel_n;
    if (nb > 0) {
      int npb = 64;
      while (npb < nb) npb <<= 1;
      for (int k = nb + tid; k < npb; k += kUpdThreads) {
        sk_l[k] = ~0ull;
        sk_v[k] = -1;
      }
      __syncthreads();
      bitonic_sort_reg<false>(nullptr, sk_l, sk_v, npb);  // ends with a barrier
    }
    // ordered compaction of the kept old nodes, in place (each thread reads its chunk first)
    constexpr int kCh = 8;  // n_old <= 8192 = 8 x kUpdThreads
    const int per_a = (n_old + kUpdThreads - 1) / kUpdThreads;
    const int a0 = min(n_old, tid * per_a), a1 = min(n_old, a0 + per_a);
    int av[kCh], acnt = 0;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
      av[k] = (a0 + k < a1) ? a_raw[a0 + k] : -1;
      acnt += av[k] >= 0;
    }
    int aex;
    const int na = block_excl_scan_fast(sm, acnt, aex);  // its barriers order the reads before the writes
#pragma unroll
    for (int k = 0; k < kCh; ++k)
      if (av[k] >= 0) a_raw[aex++] = av[k];
    __syncthreads();
    // merge the kept old run (keys lo_new[a_raw[i]]) with the new run (sk_l / sk_v) over r in [0, sel)
    const int per_o = (sel + kUpdThreads - 1) / kUpdThreads;
    const int o0 = min(sel, tid * per_o), o1 = min(sel, o0 + per_o);
    int lo_i = max(0, o0 - nb), hi_i = min(o0, na);
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (sk_l[o0 - mid - 1] < lo_new[a_raw[mid]])
        hi_i = mid;
      else
        lo_i = mid + 1;
    }
    int i = lo_i, j = o0 - lo_i;
    unsigned long long ak = i < na ? lo_new[a_raw[i]] : ~0ull;
    for (int r = o0; r < o1; ++r) {
      int pos;
      unsigned long long key;
      if (j < nb && (i >= na || sk_l[j] < ak)) {
        pos = sk_v[j];
        key = sk_l[j];
        ++j;
      } else {
        pos = a_raw[i];
        key = ak;
        ++i;
        ak = i < na ? lo_new[a_raw[i]] : ~0ull;
      }
      lex[pos] = r - ds_new[lo_depth(key)];
    }
    __syncthreads();
  } else if (n_old == 0 && 2 * ((L.V + 31) / 32) <= L.kpad * 5 && g_sort_reg) {
    // Root round: every selected node is a child of the root (depth 1, the same
    // parent), so its lex rank is the rank of its token among the selected tokens:
    // a V-bit token bitmap and a prefix popcount replace the sort (8192 keys:
    // ~150 us of bitonic network -> a few us).
    const int W = (L.V + 31) / 32;
    unsigned* bits = reinterpret_cast<unsigned*>(sk_h);  // [W] (the sort buffers span 5 kpad words)
    int* wrank = reinterpret_cast<int*>(bits + W);        // [W]: set bits in the words before
    for (int w = tid; w < W; w += kUpdThreads) bits[w] = 0u;
    __syncthreads();
    for (int pos = tid; pos < sel; pos += kUpdThreads) {
      const int tk = lo_token(lo_new[pos]);
      atomicOr(&bits[tk >> 5], 1u << (tk & 31));
    }
    __syncthreads();
    const int per_w = (W + kUpdThreads - 1) / kUpdThreads;
    const int w0 = min(W, tid * per_w), w1 = min(W, w0 + per_w);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bits[w]);
    int wex;
    block_excl_scan_fast(sm, cnt, wex);
    for (int w = w0; w < w1; ++w) {
      wrank[w] = wex;
      wex += __popc(bits[w]);
    }
    __syncthreads();
    for (int pos = tid; pos < sel; pos += kUpdThreads) {
      const int tk = lo_token(lo_new[pos]);
      lex[pos] = wrank[tk >> 5] + __popc(bits[tk >> 5] & ((1u << (tk & 31)) - 1u));
    }
    __syncthreads();
  } else {
    for (int pos = tid; pos < np2; pos += kUpdThreads) {
      sk_l[pos] = pos < sel ? lo_new[pos] : ~0ull;
      sk_v[pos] = pos;
    }
    for (int i = tid; i < 256; i += kUpdThreads) sm.depth_start[i] = 0x7fffffff;
    __syncthreads();
    if (np2 >= 64 && g_sort_reg)
      bitonic_sort_reg<false>(nullptr, sk_l, sk_v, np2);
    else
      bitonic_sort_64(sk_l, sk_v, np2);
    for (int r = tid; r < sel; r += kUpdThreads) {
      const int d = lo_depth(sk_l[r]);
      if (r == 0 || lo_depth(sk_l[r - 1]) != d) sm.depth_start[d] = r;
    }
    __syncthreads();
    for (int r = tid; r < sel; r += kUpdThreads) lex[sk_v[r]] = r - sm.depth_start[lo_depth(sk_l[r])];
    __syncthreads();
  }
  par = at<int>(ws, L.m_parent[nxt]);
  lo_arr = at<unsigned long long>(ws, L.m_lo[nxt]);
  for (int pos = tid; pos < sel; pos += kUpdThreads) {
    const unsigned long long lo = lo_arr[pos];
    const int p = par[pos];
    lo_arr[pos] = make_lo(lo_depth(lo), p < 0 ? 0 : lex[p], lo_token(lo));
  }
  __syncthreads();

  SX_TRACE(4);
  // ---- 5. threshold ----
  has_thr = sel >= K;
  th = has_thr ? (unsigned long long)__double_as_longlong(at<double>(ws, L.m_nll[nxt])[K - 1]) : 0;
  tl = has_thr ? lo_arr[K - 1] : 0;
  if (!final) {
    // merge-only slice: the batch nodes move to their new positions and lex
    // ranks (the next slice's children are keyed by them). A batch node pruned by
    // this merge (-2) gets nll = +inf: its children are worse than it, hence past
    // the new threshold, so none can survive in a later slice.
    for (int b = tid; b < c->batch_n; b += kUpdThreads) {
      const int pos = b_node[b];
      if (pos < 0) continue;  // the root
      const int np = remap[pos];
      b_node[b] = np < 0 ? -2 : np;
      if (np < 0)
        at<double>(ws, L.b_nll)[b] = CUDART_INF;
      else
        at<int>(ws, L.b_lex)[b] = lex[np];
    }
    __syncthreads();
    if (tid == 0) {
      c->cur = dst;
      c->count = sel;
      c->has_thr = has_thr;
      c->thr_nll = __longlong_as_double((long long)th);
      c->thr_lo = tl;
      c->n_surv = 0;
      at<int>(ws, L.r_aux)[0] = 0;
    }
    return;
  }
  }  // n_new > 0

  SX_TRACE(5);
  // ---- 6. next batch: first B unexpanded nodes with depth < D and key < threshold ----
  // The per-position data of the scan and of the ancestor walk is staged in
  // shared memory first (CTA 0 owns the sort buffers now): the walk follows up
  // to D dependent parent links per batch node, an L2 round trip each otherwise.
  const int per = (sel + kUpdThreads - 1) / kUpdThreads;
  const int p0 = min(sel, tid * per), p1 = min(sel, p0 + per);
  const double* nll_arr = at<double>(ws, L.m_nll[dst]);
  int* slot_arr = at<int>(ws, L.m_slot[dst]);
  int* par_s = reinterpret_cast<int*>(sk_h);  // [kpad]
  int* slot_s = par_s + L.kpad;               // [kpad] (sk_h spans 2 kpad ints)
  int* elig_s = sk_v;                         // [kpad]
  int* bnode_s = reinterpret_cast<int*>(sk_l);  // [kpad]: batch b -> position (batch_n <= sel <= kpad)
  int* bdepth_s = bnode_s + L.kpad;             // [kpad]
  // The list is sorted by key and the threshold is its K-th key, so "key <
  // threshold" is exactly "position < K - 1": no key loads. Loads are issued
  // kStg at a time per thread (independent L2 round trips).
  constexpr int kStg = 4;
  for (int base = 0; base < sel; base += kStg * kUpdThreads) {
    int sl[kStg], pr[kStg];
    unsigned long long lo[kStg];
#pragma unroll
    for (int k = 0; k < kStg; ++k) {
      const int pos = base + k * kUpdThreads + tid;
      if (pos < sel) {
        sl[k] = slot_arr[pos];
        pr[k] = par[pos];
        lo[k] = lo_arr[pos];
      }
    }
#pragma unroll
    for (int k = 0; k < kStg; ++k) {
      const int pos = base + k * kUpdThreads + tid;
      if (pos < sel) {
        par_s[pos] = pr[k];
        slot_s[pos] = sl[k];
        elig_s[pos] = sl[k] < 0 && lo_depth(lo[k]) < L.D && (!has_thr || pos < K - 1);
      }
    }
  }
  __syncthreads();
  SX_TRACE(6);
  int cnt = 0;
  for (int pos = p0; pos < p1; ++pos) cnt += elig_s[pos];
  int excl;
  const int total = block_excl_scan_fast(sm, cnt, excl);
  const int batch_n = min(total, L.B);
  const int slot_base = c->slot_next;
  int rank = excl;
  for (int pos = p0; pos < p1 && rank < batch_n; ++pos) {
    if (!elig_s[pos]) continue;
    const int b = rank++;
    const int slot = slot_base + b;
    slot_arr[pos] = slot;
    slot_s[pos] = slot;
    const unsigned long long lo = lo_arr[pos];
    const int depth = lo_depth(lo);
    bnode_s[b] = pos;
    bdepth_s[b] = depth;
    at<int>(ws, L.b_node)[b] = pos;
    at<double>(ws, L.b_nll)[b] = nll_arr[pos];
    at<int>(ws, L.b_depth)[b] = depth;
    at<int>(ws, L.b_lex)[b] = lex[pos];
    at<int>(ws, L.b_slot)[b] = slot;
    at<int>(ws, L.b_token)[b] = lo_token(lo);
    at<int>(ws, L.b_pos)[b] = c->root_slot + depth;
  }
  __syncthreads();
  SX_TRACE(7);
  // ancestor-slot lists, root first: [root_slot, slot(depth 1), ..., slot(self)]
  // (walked through the staged parent / slot tables; assembling the rows in shared
  // memory first and copying them out a warp per row measured slower)
  const int root_slot = c->root_slot;
  for (int b = tid; b < batch_n; b += kUpdThreads) {
    const int depth = bdepth_s[b];
    int* anc = at<int>(ws, L.b_anc) + b * (L.D + 1);
    int q = bnode_s[b];
    for (int k = depth; k >= 1; --k) {
      anc[k] = slot_s[q];
      q = par_s[q];
    }
    anc[0] = root_slot;
    at<int>(ws, L.b_anc_len)[b] = depth + 1;
    at<int>(ws, L.b_dense)[b] = root_slot;
  }
  SX_TRACE(8);
  // padded rows [batch_n, B): a fixed-shape draft forward (CUDA graph) may run
  // them; they write only the scratch KV slot and see just the committed prefix
  for (int b = batch_n + tid; b < L.B; b += kUpdThreads) {
    at<int>(ws, L.b_node)[b] = -1;
    at<int>(ws, L.b_token)[b] = 0;
    at<int>(ws, L.b_pos)[b] = c->root_slot;
    at<int>(ws, L.b_slot)[b] = c->pad_slot;
    at<int>(ws, L.b_anc_len)[b] = 0;
    at<int>(ws, L.b_anc)[b * (L.D + 1)] = c->pad_slot;
    at<int>(ws, L.b_dense)[b] = c->root_slot;
  }
  __syncthreads();
  SX_TRACE(9);
  if (tid == 0) {
    c->cur = dst;
    c->count = sel;
    c->has_thr = has_thr;
    c->thr_nll = __longlong_as_double((long long)th);
    c->thr_lo = tl;
    c->batch_n = batch_n;
    c->slot_next = slot_base + batch_n;
    c->n_surv = 0;
    at<int>(ws, L.r_aux)[0] = 0;  // chunked row path: empty work list for the next round
  }
}

// --------------------------------------------------------------------------
// Final tables for the target pass over the tree: row 0 = root (anchor's last
// token), row i+1 = node i. anc[row] = rows of the root path, root first, self last.
__global__ void tree_final_kernel(uint8_t* ws, TreeLayout L, int root_token, int* out_parent, int* out_token,
                                  double* out_edge, int* out_depth, int* out_slot) {
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int cur = c->cur, n = c->count;
  const int* par = at<int>(ws, L.m_parent[cur]);
  const unsigned long long* lo = at<unsigned long long>(ws, L.m_lo[cur]);
  const double* edge = at<double>(ws, L.m_edge[cur]);
  int* f_anc = at<int>(ws, L.f_anc);
  int* f_len = at<int>(ws, L.f_anc_len);
  int* f_depth = at<int>(ws, L.f_depth);
  int* f_tok = at<int>(ws, L.f_token);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += gridDim.x * blockDim.x) {
    int* anc = f_anc + (long long)r * (L.D + 1);
    if (r == 0) {
      anc[0] = 0;
      f_len[0] = 1;
      f_depth[0] = 0;
      f_tok[0] = root_token;
      continue;
    }
    const int i = r - 1;
    const int depth = lo_depth(lo[i]);
    f_depth[r] = depth;
    f_tok[r] = lo_token(lo[i]);
    f_len[r] = depth + 1;
    int q = i;
    for (int k = depth; k >= 1; --k) {
      anc[k] = q + 1;
      q = par[q];
    }
    anc[0] = 0;
    if (out_parent) out_parent[i] = par[i];
    if (out_token) out_token[i] = lo_token(lo[i]);
    if (out_edge) out_edge[i] = edge[i];
    if (out_depth) out_depth[i] = depth;
    if (out_slot) out_slot[i] = at<int>(ws, L.m_slot[cur])[i];
  }
}

// --------------------------------------------------------------------------
// Exact table models on the GPU (MarkovModel / TabularModel, models.py:77-151):
// rows for tree nodes. node_ids[i] = position in the current materialized list,
// or -1 for the root (the anchor itself). ctx0 = anchor's last `order` tokens,
// left-padded with 0 (models.py:127-129).
__global__ void markov_rows_kernel(const double* __restrict__ table, int V, int order, const int* ctx0,
                                   uint8_t* ws, TreeLayout L, const int* node_ids, int n_nodes, int from_batch,
                                   double* out, long long ld) {
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  const int i = blockIdx.x;
  const int cnt = from_batch ? c->batch_n : n_nodes;
  if (i >= cnt) return;
  __shared__ long long row_idx;
  if (threadIdx.x == 0) {
    const int cur = c->cur;
    const int* par = at<int>(ws, L.m_parent[cur]);
    const unsigned long long* lo = at<unsigned long long>(ws, L.m_lo[cur]);
    int node = from_batch ? at<int>(ws, L.b_node)[i] : node_ids[i];
    int toks[64];
    int nt = 0;
    while (node >= 0 && nt < order) {
      toks[nt++] = lo_token(lo[node]);
      node = par[node];
    }
    // context = (ctx0 + path)[-order:]
    long long idx = 0;
    for (int k = 0; k < order; ++k) {
      const int pos_from_end = order - 1 - k;  // 0 = last token
      const int t = pos_from_end < nt ? toks[pos_from_end] : ctx0[order - 1 - (pos_from_end - nt)];
      idx = idx * V + t;
    }
    row_idx = idx;
  }
  __syncthreads();
  const double* src = table + row_idx * V;
  double* dst = out + (long long)i * ld;
  for (int v = threadIdx.x; v < V; v += blockDim.x) dst[v] = src[v];
}

// --------------------------------------------------------------------------
// KB1/KB2: beam search (build_beam, pkg/src/speckit/tree.py:330-380).
// KB1, one CTA per beam row: every token with q > 0 gets nll = beam_nll - log q
// (canonical log), the row's candidates are radix-sorted by (nll, token) and
// the first k kept (no other candidate of the row can reach the global top k:
// its path prefix is shared). KB2, one CTA: the nb x k survivors sorted by
// (nll, lex rank of the beam path, token) -- the reference's (nll, path) order
// for equal-length paths -- and the first beam_size returned.
__global__ void __launch_bounds__(kRowThreads) beam_row_topk_kernel(const double* q, long long ldq, int V,
                                                                     const double* beam_nll, int k,
                                                                     unsigned long long* keys, int* idx,
                                                                     unsigned long long* keys2, int* idx2,
                                                                     double* c_nll, double* c_edge, int* c_tok,
                                                                     int* c_cnt) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  const int b = blockIdx.x;
  const double* row = q + (long long)b * ldq;
  const long long o = (long long)b * V;
  const double bn = beam_nll[b];
  int valid = 0;
  for (int v = threadIdx.x; v < V; v += kRowThreads) {
    const double p = row[v];
    unsigned long long key = ~0ULL;
    if (p > 0.0) {
      key = (unsigned long long)__double_as_longlong(dsub(bn, sx_log(p)));
      ++valid;
    }
    keys[o + v] = key;
    idx[o + v] = v;
  }
  __threadfence_block();
  __syncthreads();
  block_radix_sort(sm, keys + o, idx + o, keys2 + o, idx2 + o, V, 8);  // 8 passes: result in keys/idx
  // count of valid entries = block sum of `valid`
  sm.redi[threadIdx.x] = valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kRowThreads; ++i) tot += sm.redi[i];
    sm.redi[0] = tot;
  }
  __syncthreads();
  const int cnt = min(k, sm.redi[0]);
  for (int i = threadIdx.x; i < cnt; i += kRowThreads) {
    const int tok = idx[o + i];
    const double nll = __longlong_as_double((long long)keys[o + i]);
    c_nll[(long long)b * k + i] = nll;
    c_edge[(long long)b * k + i] = sx_log(row[tok]);
    c_tok[(long long)b * k + i] = tok;
  }
  if (threadIdx.x == 0) c_cnt[b] = cnt;
}

constexpr int kBeamSortMax = 8192;

__global__ void __launch_bounds__(1024) beam_select_kernel(int nb, int k, const int* beam_rank, const double* c_nll,
                                                          const double* c_edge, const int* c_tok, const int* c_cnt,
                                                          int beam_size, int* out_n, double* out_nll,
                                                          double* out_edge, int* out_beam, int* out_tok) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int total = nb * k;
  int n = 1;
  while (n < total) n <<= 1;
  unsigned long long* kh = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* kl = kh + n;
  int* kv = reinterpret_cast<int*>(kl + n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int b = i / k, j = i % k;
    if (i < total && j < c_cnt[b]) {
      kh[i] = (unsigned long long)__double_as_longlong(c_nll[i]);
      kl[i] = ((unsigned long long)(unsigned)beam_rank[b] << 32) | (unsigned)c_tok[i];
      kv[i] = i;
    } else {
      kh[i] = ~0ULL;
      kl[i] = ~0ULL;
      kv[i] = -1;
    }
  }
  __syncthreads();
  bitonic_sort_128(kh, kl, kv, n);
  __shared__ int s_n;
  if (threadIdx.x == 0) {
    int c = 0;
    while (c < beam_size && c < n && kv[c] >= 0) ++c;
    s_n = c;
    *out_n = c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_n; i += blockDim.x) {
    const int src = kv[i];
    out_nll[i] = c_nll[src];
    out_edge[i] = c_edge[src];
    out_beam[i] = src / k;
    out_tok[i] = c_tok[src];
  }
}

}  // namespace sx

using namespace sx;

extern "C" long long sx_beam_scratch_bytes(int nb, int V) {
  const long long e = (long long)nb * V;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  return 2 * al(8 * e) + 2 * al(4 * e);
}

extern "C" int sx_beam_step(const double* q, long long ldq, int V, int nb, const double* beam_nll,
                            const int* beam_rank, int beam_size, void* scratch, double* c_nll, double* c_edge,
                            int* c_tok, int* c_cnt, int* out_n, double* out_nll, double* out_edge, int* out_beam,
                            int* out_tok, cudaStream_t stream) {
  if (nb < 1 || V < 2 || beam_size < 1) return arg_error("beam_step: need nb >= 1, V >= 2, beam_size >= 1");
  if ((long long)nb * beam_size > kBeamSortMax)
    return arg_error("beam_step: %d beams x beam_size %d exceed the %d-entry single-CTA sort", nb, beam_size,
                     kBeamSortMax);
  if (int st = ensure_smem_attr((const void*)beam_row_topk_kernel, (int)sizeof(RowSmem))) return st;
  if (int st = ensure_smem_attr((const void*)beam_select_kernel, kBeamSortMax * 20)) return st;
  const long long e = (long long)nb * V;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  uint8_t* s = reinterpret_cast<uint8_t*>(scratch);
  unsigned long long* k1 = reinterpret_cast<unsigned long long*>(s);
  unsigned long long* k2 = reinterpret_cast<unsigned long long*>(s + al(8 * e));
  int* i1 = reinterpret_cast<int*>(s + 2 * al(8 * e));
  int* i2 = reinterpret_cast<int*>(s + 2 * al(8 * e) + al(4 * e));
  const int k = beam_size;
  beam_row_topk_kernel<<<nb, kRowThreads, sizeof(RowSmem), stream>>>(q, ldq, V, beam_nll, k, k1, i1, k2, i2, c_nll,
                                                                       c_edge, c_tok, c_cnt);
  SX_CHECK_LAUNCH("beam_row_topk_kernel");
  int n = 1;
  while (n < nb * k) n <<= 1;
  const size_t smem = (size_t)n * 20;
  beam_select_kernel<<<1, 1024, smem, stream>>>(nb, k, beam_rank, c_nll, c_edge, c_tok, c_cnt, beam_size, out_n,
                                                out_nll, out_edge, out_beam, out_tok);
  SX_CHECK_LAUNCH("beam_select_kernel");
  return SX_OK;
}

static long long g_survivor_cap = 0;  // sx_tree_set_survivor_cap: 0 = default_survivor_cap (tests force overflows)

static TreeLayout host_layout(int K, int B, int V, int D) {
  long long cap = g_survivor_cap > 0 ? g_survivor_cap : default_survivor_cap(K, B, V);
  if (cap < V) cap = V;  // a single row's candidates always fit: the sliced retry makes progress
  return tree_layout(K, B, V, D, cap);
}

extern "C" int sx_tree_set_survivor_cap(long long cap) {
  if (cap < 0) return arg_error("survivor cap must be >= 0 (0 = default)");
  g_survivor_cap = cap;
  return SX_OK;
}

extern "C" long long sx_tree_survivor_cap(int K, int B, int V, int D) {
  if (K < 1 || B < 1 || V < 2 || D < 1 || D > 250) return -1;
  return host_layout(K, B, V, D).cap;
}

static size_t upd_smem_bytes(const TreeLayout& L) {
  return ((sizeof(UpdSmem) + 15) & ~size_t(15)) + (size_t)L.kpad * (8 + 8 + 4) + 64;
}

extern "C" long long sx_tree_workspace_bytes(int K, int B, int V, int D) {
  if (K < 1 || B < 1 || V < 2 || D < 1 || D > 250) return -1;
  return host_layout(K, B, V, D).total;
}

extern "C" int sx_tree_offsets(int K, int B, int V, int D, long long* out, int n) {
  TreeLayout L = host_layout(K, B, V, D);
  const long long vals[] = {L.ctl,   L.b_node,    L.b_nll, L.b_depth,   L.b_lex,   L.b_slot,  L.b_token, L.b_anc,
                            L.b_anc_len, L.f_anc, L.f_anc_len, L.f_depth, L.f_token, L.w_rows, L.b_pos, L.b_dense, L.total, L.r_aux};
  const int m = (int)(sizeof(vals) / sizeof(vals[0]));
  for (int i = 0; i < n && i < m; ++i) out[i] = vals[i];
  return m;
}

static int check_tree_args(int K, int B, int V, int D) {
  if (K < 1 || B < 1 || V < 2 || D < 1) return arg_error("tree: need K, B, D >= 1 and V >= 2");
  if (K > 8192) return arg_error("tree: budget K=%d exceeds the 8192 single-CTA select/sort capacity", K);
  if (D > 250) return arg_error("tree: max_depth %d > 250", D);
  if (V > 262144) return arg_error("tree: vocab %d > 262144", V);
  return SX_OK;
}

extern "C" int sx_tree_begin(void* ws, int K, int B, int V, int D, int root_slot, int pad_slot, cudaStream_t stream) {
  int st = check_tree_args(K, B, V, D);
  if (st) return st;
  TreeLayout L = host_layout(K, B, V, D);
  tree_begin_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<uint8_t*>(ws), L, root_slot, pad_slot);
  SX_CHECK_LAUNCH("tree_begin_kernel");
  return SX_OK;
}

// SX_TREE_PDL=0: ordinary stream order for the chunked row path and the update (A/B)
static const int g_tree_pdl = getenv("SX_TREE_PDL") ? atoi(getenv("SX_TREE_PDL")) : 1;

template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_tree_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// SX_TREE_FUSED_EXACT=0: separate sum and score kernels (A/B)
static const int g_tree_fused_exact = getenv("SX_TREE_FUSED_EXACT") ? atoi(getenv("SX_TREE_FUSED_EXACT")) : 1;

static int g_tree_unfused = 0;  // sx_tree_set_impl: 1 = the two-kernel row_stats + score path (A/B)

extern "C" int sx_tree_set_impl(int unfused) {
  if (unfused < 0 || unfused > 1) return arg_error("tree impl %d (0 fused rows kernel, 1 row_stats + score)", unfused);
  g_tree_unfused = unfused;
  return SX_OK;
}

extern "C" int sx_tree_round(void* ws, int K, int B, int V, int D, const void* rows, int row_kind, long long ld,
                             int score_mode, double temperature, double top_p, int* host_ctl, cudaStream_t stream) {
  return sx_tree_round_rows(ws, K, B, V, D, rows, row_kind, ld, score_mode, temperature, top_p, 0, -1, 1, host_ctl,
                            stream);
}

extern "C" int sx_tree_round_rows(void* ws, int K, int B, int V, int D, const void* rows, int row_kind, long long ld,
                                  int score_mode, double temperature, double top_p, int r0, int r1, int final,
                                  int* host_ctl, cudaStream_t stream) {
  int st = check_tree_args(K, B, V, D);
  if (st) return st;
  if (row_kind != SX_ROWS_LOGITS_F32 && row_kind != SX_ROWS_PROBS_F64) return arg_error("tree: bad row kind");
  if (ld < V) return arg_error("tree: row stride %lld < V %d", ld, V);
  if (r0 < 0 || r0 >= B || (r1 >= 0 && r1 <= r0) || r1 > B) return arg_error("tree: bad row range [%d, %d)", r0, r1);
  TreeLayout L = host_layout(K, B, V, D);
  const int nrows = (r1 < 0 ? B : r1) - r0;  // grid bound; the kernels clip to batch_n
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  if (int st = ensure_smem_attr((const void*)tree_update_kernel, 227 * 1024)) return st;
  if (int st = ensure_smem_attr((const void*)tree_warp_rows_kernel, (int)sizeof(RowSmem))) return st;
  if (int st = ensure_smem_attr((const void*)tree_argmax_score_kernel, (int)sizeof(RowSmem))) return st;
  if (score_mode == SX_SCORE_ARGMAX) {
    tree_argmax_score_kernel<<<nrows, kRowThreads, sizeof(RowSmem), stream>>>(w, L, rows, row_kind, ld, r0, r1);
    SX_CHECK_LAUNCH("tree_argmax_score_kernel");
  } else if (score_mode == SX_SCORE_WARP) {
    tree_warp_rows_kernel<<<L.wsc, kRowThreads, sizeof(RowSmem), stream>>>(w, L, rows, row_kind, ld, temperature,
                                                                         top_p, r0, r1);
    SX_CHECK_LAUNCH("tree_warp_rows_kernel");
    dim3 grid((V + 255) / 256 < 64 ? (V + 255) / 256 : 64, nrows);
    tree_score_kernel<<<grid, 256, 0, stream>>>(w, L, nullptr, -1, V, r0, r1);
    SX_CHECK_LAUNCH("tree_score_kernel");
  } else if (score_mode == SX_SCORE_RAW && row_kind == SX_ROWS_LOGITS_F32 && !g_tree_unfused) {
    // persistent grids of (row, chunk) units, sized to the resident CTAs
    static int occ[3] = {0, 0, 0};
    if (!occ[0]) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], tree_rows_max_kernel<2>, kMaxThreads, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], tree_rows_sum_kernel, kRowThreads, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[2], tree_rows_score_kernel, kRowThreads, 0);
      for (int& o : occ) o = o < 1 ? 1 : o;
    }
    const long long ua = (long long)nrows * ((V + kRowChunkA - 1) / kRowChunkA);
    const long long ub = (long long)nrows * ((V + kRowChunkB - 1) / kRowChunkB);
    auto grid_of = [&](long long units, int o) { return (int)(units < (long long)o * kNumSMs ? units : (long long)o * kNumSMs); };
    const float* z = reinterpret_cast<const float*>(rows);
    // vec4: 2 = pipelined batch-max loop, 1 = per-element online loop (SX_TREE_MAX_PIPE=0, A/B), 0 = scalar
    static const int pipe = getenv("SX_TREE_MAX_PIPE") ? atoi(getenv("SX_TREE_MAX_PIPE")) : 1;
    const int vec4 = ((V % 4 == 0) && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(rows) & 15) == 0))
                         ? (pipe == 2 ? 3 : (pipe ? 2 : 1))
                         : 0;
    if (vec4 == 3) {
      static int occ3 = 0;
      if (!occ3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, tree_rows_max_kernel<3>, kMaxThreads, 0);
      tree_rows_max_kernel<3><<<grid_of(ua, occ3 < 1 ? 1 : occ3), kMaxThreads, 0, stream>>>(w, L, z, ld, r0, r1);
    } else if (vec4 == 2)
      tree_rows_max_kernel<2><<<grid_of(ua, occ[0]), kMaxThreads, 0, stream>>>(w, L, z, ld, r0, r1);
    else if (vec4 == 1)
      tree_rows_max_kernel<1><<<grid_of(ua, occ[0]), kMaxThreads, 0, stream>>>(w, L, z, ld, r0, r1);
    else
      tree_rows_max_kernel<0><<<grid_of(ua, occ[0]), kMaxThreads, 0, stream>>>(w, L, z, ld, r0, r1);
    SX_CHECK_LAUNCH("tree_rows_max_kernel");
    // sum, score and the update are launched with programmatic stream serialization:
    // each grid becomes resident while its predecessor drains and waits in
    // griddepcontrol.wait (full completion + memory flush), hiding the launch gaps
    if (g_tree_fused_exact) {
      static int occx = 0;
      if (!occx) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occx, tree_rows_exact_kernel, kRowThreads, 0);
        if (occx < 1) occx = 1;
      }
      // The score units spin on flags set by sum units of other CTAs, so every CTA
      // must be resident at once: grid <= the resident capacity, and a cooperative
      // launch makes the co-residency a guarantee even when other work (another
      // engine's stream) shares the GPU.
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid_of(ub, occx));
      cfg.blockDim = dim3(kRowThreads);
      cfg.stream = stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = g_tree_pdl;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      cudaLaunchKernelEx(&cfg, tree_rows_exact_kernel, w, L, z, ld);
      SX_CHECK_LAUNCH("tree_rows_exact_kernel");
    } else {
      launch_pdl(tree_rows_sum_kernel, dim3(grid_of(ub, occ[1])), dim3(kRowThreads), 0, stream, w, L, z, ld);
      SX_CHECK_LAUNCH("tree_rows_sum_kernel");
      launch_pdl(tree_rows_score_kernel, dim3(grid_of(ub, occ[2])), dim3(kRowThreads), 0, stream, w, L, z, ld);
      SX_CHECK_LAUNCH("tree_rows_score_kernel");
    }
  } else if (score_mode == SX_SCORE_RAW) {
    if (row_kind == SX_ROWS_LOGITS_F32) {
      tree_row_stats_kernel<<<nrows, kRowThreads, 0, stream>>>(w, L, reinterpret_cast<const float*>(rows), ld, r0, r1);
      SX_CHECK_LAUNCH("tree_row_stats_kernel");
    }
    dim3 grid((V + 255) / 256 < 64 ? (V + 255) / 256 : 64, nrows);
    tree_score_kernel<<<grid, 256, 0, stream>>>(w, L, rows, row_kind, ld, r0, r1);
    SX_CHECK_LAUNCH("tree_score_kernel");
  } else {
    return arg_error("tree: bad score mode %d", score_mode);
  }
  const size_t smem = upd_smem_bytes(L);
  if (smem > 227 * 1024) return arg_error("tree: update needs %zu B of shared memory", smem);
  static const int sort_reg_init = [] {
    const int v = getenv("SX_TREE_SORT_REG") ? atoi(getenv("SX_TREE_SORT_REG")) : 1;
    if (v != 1) cudaMemcpyToSymbol(g_sort_reg, &v, sizeof(int));
    const int m = getenv("SX_TREE_MERGE") ? atoi(getenv("SX_TREE_MERGE")) : 1;
    if (m != 1) cudaMemcpyToSymbol(g_update_merge, &m, sizeof(int));
    return v;
  }();
  (void)sort_reg_init;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kUpdCluster);
    cfg.blockDim = dim3(kUpdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kUpdCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = g_tree_pdl;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, tree_update_kernel, w, L, final);
  }
  SX_CHECK_LAUNCH("tree_update_kernel");
  if (host_ctl) {
    cudaError_t e = cudaMemcpyAsync(host_ctl, w + L.ctl, sizeof(TreeCtl), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return cuda_status(e, "sx_tree_round: ctl readback");
  }
  return SX_OK;
}

__global__ void tree_clear_err_kernel(uint8_t* ws, TreeLayout L) {
  TreeCtl* c = at<TreeCtl>(ws, L.ctl);
  c->err = 0;
  c->n_surv = 0;
  at<int>(ws, L.r_aux)[0] = 0;
}

extern "C" int sx_tree_clear_overflow(void* ws, int K, int B, int V, int D, cudaStream_t stream) {
  int st = check_tree_args(K, B, V, D);
  if (st) return st;
  tree_clear_err_kernel<<<1, 1, 0, stream>>>(reinterpret_cast<uint8_t*>(ws), host_layout(K, B, V, D));
  SX_CHECK_LAUNCH("tree_clear_err_kernel");
  return SX_OK;
}

extern "C" int sx_tree_finalize(void* ws, int K, int B, int V, int D, int root_token, int* out_parent, int* out_token,
                                double* out_edge, int* out_depth, int* out_slot, cudaStream_t stream) {
  int st = check_tree_args(K, B, V, D);
  if (st) return st;
  TreeLayout L = host_layout(K, B, V, D);
  tree_final_kernel<<<(K + 256) / 256, 256, 0, stream>>>(reinterpret_cast<uint8_t*>(ws), L, root_token, out_parent,
                                                          out_token, out_edge, out_depth, out_slot);
  SX_CHECK_LAUNCH("tree_final_kernel");
  return SX_OK;
}

extern "C" int sx_markov_rows(const double* table, int V, int order, const int* ctx0, void* ws, int K, int B, int D,
                              const int* node_ids, int n_nodes, int from_batch, double* out, long long ld,
                              cudaStream_t stream) {
  int st = check_tree_args(K, B, V, D);
  if (st) return st;
  if (order < 0 || order > 64) return arg_error("markov: order %d out of range", order);
  TreeLayout L = host_layout(K, B, V, D);
  const int grid = from_batch ? B : n_nodes;
  if (grid <= 0) return SX_OK;
  markov_rows_kernel<<<grid, 128, 0, stream>>>(table, V, order, ctx0, reinterpret_cast<uint8_t*>(ws), L, node_ids,
                                               n_nodes, from_batch, out, ld);
  SX_CHECK_LAUNCH("markov_rows_kernel");
  return SX_OK;
}
