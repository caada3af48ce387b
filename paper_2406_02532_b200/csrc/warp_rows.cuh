// Block-level (256 threads, one CTA per row) canonical float64 row kernels:
// softmax, temperature / nucleus warp (apply_warp, pkg/src/speckit/sampling.py:66-98)
// and the inverse-CDF sample (sampling.py:101-113).
//
// Canonical arithmetic (shared definition with oracle/oxmath.c):
//   sum     : lane j of 256 adds elements j, j+256, ... in order from +0.0, then
//             the 256 lane sums are combined by a halving tree;
//   cumsum  : blocks of 256 consecutive elements (in scan order), sequential
//             inside a block, block totals chained sequentially;
//   log/exp : sx_log / sx_exp (sxmath.cuh).
// The nucleus sort orders by (probability desc, token id asc) with a stable
// LSD radix sort in global scratch (keys: transformed fp32 logit or fp64 prob).
#pragma once
#include "common.cuh"
#include "sxmath.cuh"

namespace sx {

constexpr int kRowThreads = 256;

struct RowSmem {
  double red[kRowThreads];
  float redf[kRowThreads];
  int redi[kRowThreads];
  unsigned short hist[256][kRowThreads];  // radix counts [bin][thread]
  int bin_base[256];
  int grp_base[256][kRowThreads / 32];
  double blk_prefix[1024];
  int cut;
};

struct RowSmemLite {
  double red[kRowThreads];
  float redf[kRowThreads];
  int redi[kRowThreads];
};

// ---- reductions (blockDim == 256) -----------------------------------------
template <class SM>
SX_DEV double block_canon_sum(SM& sm, double lane_acc) {
  const int t = threadIdx.x;
  sm.red[t] = lane_acc;
  __syncthreads();
  for (int w = kRowThreads / 2; w >= 1; w >>= 1) {
    if (t < w) sm.red[t] = dadd(sm.red[t], sm.red[t + w]);
    __syncthreads();
  }
  const double s = sm.red[0];
  __syncthreads();
  return s;
}

template <class SM>
SX_DEV float block_max_f(SM& sm, float v) {
  const int t = threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  if ((t & 31) == 0) sm.redf[t >> 5] = v;
  __syncthreads();
  if (t < 32) {
    float x = t < kRowThreads / 32 ? sm.redf[t] : -CUDART_INF_F;
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffff, x, o));
    if (t == 0) sm.redf[0] = x;
  }
  __syncthreads();
  const float r = sm.redf[0];
  __syncthreads();
  return r;
}

// argmax with lowest index on ties; values compared as doubles.
template <class SM>
SX_DEV int block_argmax(SM& sm, double v, int idx) {
  const int t = threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffff, v, o);
    int oi = __shfl_xor_sync(0xffffffff, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if ((t & 31) == 0) {
    sm.red[t >> 5] = v;
    sm.redi[t >> 5] = idx;
  }
  __syncthreads();
  if (t == 0) {
    double bv = sm.red[0];
    int bi = sm.redi[0];
    for (int w = 1; w < kRowThreads / 32; ++w)
      if (sm.red[w] > bv || (sm.red[w] == bv && sm.redi[w] < bi)) {
        bv = sm.red[w];
        bi = sm.redi[w];
      }
    sm.redi[0] = bi;
  }
  __syncthreads();
  const int r = sm.redi[0];
  __syncthreads();
  return r;
}

template <class SM>
SX_DEV int block_min_i(SM& sm, int v) {
  const int t = threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffff, v, o));
  if ((t & 31) == 0) sm.redi[t >> 5] = v;
  __syncthreads();
  if (t == 0) {
    int b = sm.redi[0];
    for (int w = 1; w < kRowThreads / 32; ++w) b = min(b, sm.redi[w]);
    sm.redi[0] = b;
  }
  __syncthreads();
  const int r = sm.redi[0];
  __syncthreads();
  return r;
}

template <class SM>
SX_DEV int block_max_i(SM& sm, int v) {
  const int t = threadIdx.x;
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffff, v, o));
  if ((t & 31) == 0) sm.redi[t >> 5] = v;
  __syncthreads();
  if (t == 0) {
    int b = sm.redi[0];
    for (int w = 1; w < kRowThreads / 32; ++w) b = max(b, sm.redi[w]);
    sm.redi[0] = b;
  }
  __syncthreads();
  const int r = sm.redi[0];
  __syncthreads();
  return r;
}

// ---- softmax statistics -------------------------------------------------------
// m = max z; S = canonical sum of sx_exp(((double)z - m) * scale) (scale = 1/T or 1)
template <class SM>
SX_DEV void row_stats(SM& sm, const float* z, int V, double scale, bool use_scale, float& m, double& S) {
  float mx = -CUDART_INF_F;
  for (int v = threadIdx.x; v < V; v += kRowThreads) mx = fmaxf(mx, z[v]);
  m = block_max_f(sm, mx);
  double acc = 0.0;
  for (int v = threadIdx.x; v < V; v += kRowThreads) {
    double a = dsub((double)z[v], (double)m);
    if (use_scale) a = dmul(a, scale);
    acc = dadd(acc, sx_exp(a));
  }
  S = block_canon_sum(sm, acc);
}

template <class SM>
SX_DEV void row_stats_lite(SM& sm, const float* z, int V, float& m, double& S) {
  row_stats(sm, z, V, 1.0, false, m, S);
}

// ---- stable LSD radix sort of (key, idx) pairs in global scratch -----------------
// keys are sorted ascending; `nbytes` 8-bit passes over the low bytes of the key.
SX_DEV void block_radix_sort(RowSmem& sm, unsigned long long* keys, int* idx, unsigned long long* keys2, int* idx2,
                             int n, int nbytes) {
  const int t = threadIdx.x;
  const int chunk = (n + kRowThreads - 1) / kRowThreads;
  const int b0 = min(n, t * chunk), b1 = min(n, b0 + chunk);
  for (int pass = 0; pass < nbytes; ++pass) {
    const int sh = 8 * pass;
    for (int b = 0; b < 256; ++b) sm.hist[b][t] = 0;
    for (int i = b0; i < b1; ++i) sm.hist[(keys[i] >> sh) & 255][t]++;
    __syncthreads();
    // thread t owns bin t: exclusive offsets inside groups of 32 threads
    // (<= 32 * chunk, fits u16) plus 32-bit group bases.
    int tot = 0;
    for (int g = 0; g < kRowThreads / 32; ++g) {
      sm.grp_base[t][g] = tot;
      int run = 0;
      for (int u = g * 32; u < g * 32 + 32; ++u) {
        const int c = sm.hist[t][u];
        sm.hist[t][u] = (unsigned short)run;
        run += c;
      }
      tot += run;
    }
    sm.redi[t] = tot;
    __syncthreads();
    if (t == 0) {
      int run = 0;
      for (int b = 0; b < 256; ++b) {
        sm.bin_base[b] = run;
        run += sm.redi[b];
      }
    }
    __syncthreads();
    for (int i = b0; i < b1; ++i) {
      const int d = (keys[i] >> sh) & 255;
      const int pos = sm.bin_base[d] + sm.grp_base[d][t >> 5] + sm.hist[d][t];
      sm.hist[d][t]++;
      keys2[pos] = keys[i];
      idx2[pos] = idx[i];
    }
    __syncthreads();
    // swap buffers
    unsigned long long* tk = keys;
    keys = keys2;
    keys2 = tk;
    int* ti = idx;
    idx = idx2;
    idx2 = ti;
    __threadfence_block();
    __syncthreads();
  }
}

// ---- canonical cumsum search ------------------------------------------------------
// Over x[order[i]] (or x[i] when order == nullptr), i in [0, n): returns the first i
// whose canonical inclusive prefix sum satisfies `ge ? (c >= target) : (c > target)`,
// or n if none. Also returns the total (last prefix) through *total when non-null.
SX_DEV int block_cumsum_search(RowSmem& sm, const double* x, const int* order, int n, double target, bool ge,
                               double* total_out) {
  const int t = threadIdx.x;
  const int nblk = (n + 255) / 256;  // <= 1024 supported
  // block totals
  for (int b = t; b < nblk; b += kRowThreads) {
    double local = 0.0;
    const int e = min(n, (b + 1) * 256);
    for (int i = b * 256; i < e; ++i) local = dadd(local, x[order ? order[i] : i]);
    sm.blk_prefix[b] = local;
  }
  __syncthreads();
  if (t == 0) {
    double run = 0.0;
    for (int b = 0; b < nblk; ++b) {
      const double l = sm.blk_prefix[b];
      sm.blk_prefix[b] = run;  // incoming prefix
      run = dadd(run, l);
    }
    sm.red[0] = run;
  }
  __syncthreads();
  const double total = sm.red[0];
  int found = n;
  for (int b = t; b < nblk; b += kRowThreads) {
    const double pre = sm.blk_prefix[b];
    double local = 0.0;
    const int e = min(n, (b + 1) * 256);
    for (int i = b * 256; i < e; ++i) {
      local = dadd(local, x[order ? order[i] : i]);
      const double c = dadd(pre, local);
      if (ge ? (c >= target) : (c > target)) {
        found = min(found, i);
        break;
      }
    }
  }
  __syncthreads();
  const int r = block_min_i(sm, found);
  if (total_out) *total_out = total;
  return r;
}

// ---- full canonical warp of one row into out[V] (fp64) ----------------------------
// mode: z != nullptr -> from fp32 logits; else from fp64 probabilities p.
// temperature == 0 -> one-hot argmax (lowest id).
SX_DEV void warp_row(RowSmem& sm, const float* z, const double* p, int V, double temperature, double top_p,
                     double* out, unsigned long long* k1, int* i1, unsigned long long* k2, int* i2) {
  const int t = threadIdx.x;
  if (temperature == 0.0) {
    double bv = -CUDART_INF;
    int bi = 0x7fffffff;
    for (int v = t; v < V; v += kRowThreads) {
      const double x = z ? (double)z[v] : p[v];
      if (x > bv) {
        bv = x;
        bi = v;
      }
    }
    const int best = block_argmax(sm, bv, bi);
    for (int v = t; v < V; v += kRowThreads) out[v] = (v == best) ? 1.0 : 0.0;
    __syncthreads();
    return;
  }
  const bool scale = temperature != 1.0;
  const double invT = 1.0 / temperature;
  if (z) {
    float m;
    double S;
    row_stats(sm, z, V, invT, scale, m, S);
    for (int v = t; v < V; v += kRowThreads) {
      double a = dsub((double)z[v], (double)m);
      if (scale) a = dmul(a, invT);
      out[v] = ddiv(sx_exp(a), S);
    }
  } else if (scale) {
    double acc = 0.0;
    for (int v = t; v < V; v += kRowThreads) {
      const double e = p[v] > 0.0 ? sx_exp(dmul(sx_log(p[v]), invT)) : 0.0;
      out[v] = e;
      acc = dadd(acc, e);
    }
    const double S = block_canon_sum(sm, acc);
    for (int v = t; v < V; v += kRowThreads) out[v] = ddiv(out[v], S);
  } else {
    for (int v = t; v < V; v += kRowThreads) out[v] = p[v];
  }
  __syncthreads();
  if (top_p < 1.0) {
    // sort (prob desc, id asc): ascending sort of inverted order-preserving keys
    for (int v = t; v < V; v += kRowThreads) {
      unsigned long long key;
      if (z) {
        const unsigned u = __float_as_uint(z[v]);
        const unsigned ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        key = (unsigned long long)(~ord);
      } else {
        key = ~(unsigned long long)__double_as_longlong(out[v]);
      }
      k1[v] = key;
      i1[v] = v;
    }
    __threadfence_block();
    __syncthreads();
    const int nbytes = z ? 4 : 8;
    block_radix_sort(sm, k1, i1, k2, i2, V, nbytes);
    const int* order = (nbytes & 1) ? i2 : i1;  // result lands in i1 after an even number of passes
    const int cut0 = block_cumsum_search(sm, out, order, V, top_p - 1e-9, true, nullptr);
    const int cut = cut0 >= V ? V - 1 : cut0;
    for (int i = cut + 1 + t; i < V; i += kRowThreads) out[order[i]] = 0.0;
    __threadfence_block();
    __syncthreads();
    double acc = 0.0;
    for (int v = t; v < V; v += kRowThreads) acc = dadd(acc, out[v]);
    const double S = block_canon_sum(sm, acc);
    for (int v = t; v < V; v += kRowThreads) out[v] = ddiv(out[v], S);
    __threadfence_block();
    __syncthreads();
  }
}

// inverse-CDF sample over ascending ids of a warped row (sampling.py:101-113)
SX_DEV int sample_row(RowSmem& sm, const double* w, int V, double u) {
  double total;
  // find first i with cdf[i] > u * cdf[-1]: need the total first
  {
    const int t = threadIdx.x;
    const int nblk = (V + 255) / 256;
    for (int b = t; b < nblk; b += kRowThreads) {
      double local = 0.0;
      const int e = min(V, (b + 1) * 256);
      for (int i = b * 256; i < e; ++i) local = dadd(local, w[i]);
      sm.blk_prefix[b] = local;
    }
    __syncthreads();
    if (t == 0) {
      double run = 0.0;
      for (int b = 0; b < nblk; ++b) run = dadd(run, sm.blk_prefix[b]);
      sm.red[0] = run;
    }
    __syncthreads();
    total = sm.red[0];
    __syncthreads();
  }
  int tok = block_cumsum_search(sm, w, nullptr, V, dmul(u, total), false, nullptr);
  if (tok >= V || w[tok] == 0.0) {
    int best = -1;
    for (int v = threadIdx.x; v < V; v += kRowThreads)
      if (w[v] != 0.0) best = max(best, v);
    tok = block_max_i(sm, best);
    if (tok < 0) tok = 0;
  }
  return tok;
}

}  // namespace sx
