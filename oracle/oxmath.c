/*
 * oxmath.c -- TEST INFRASTRUCTURE (the CPU oracle's float64 kernels).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this. It is the checker, never the product path.
 *
 * What it restates:
 *  - the float64 scoring pipeline of the reference: probabilities from logits,
 *    temperature / nucleus warp (pkg/src/speckit/sampling.py:66-98), edge
 *    log-probs `np.log(p)` (pkg/src/speckit/tree.py:230-232) and the inverse-CDF
 *    sample (pkg/src/speckit/sampling.py:101-113);
 *  - with ONE documented deviation from numpy: elementary functions and
 *    summation orders are fixed ("canonical") instead of numpy's
 *    CPU-dispatch-dependent SIMD log/exp and pairwise sums:
 *      log, exp  : fdlibm __ieee754_log / __ieee754_exp (< 1 ulp), evaluated
 *                  with non-contracted IEEE ops (compile with -ffp-contract=off);
 *      row sum   : 256 strided lanes summed sequentially, then a halving tree;
 *      cumsum    : blocks of 256 in scan order, block totals chained
 *                  sequentially, sequential within a block.
 *    The B200 kernels evaluate the identical expression trees, so GPU and
 *    oracle agree bit-for-bit; against numpy the values differ by <= a few ulp
 *    and tree topology / tokens agree except on documented near-ties (see
 *    tests/test_oracle_pinned.py and DESIGN.md "Parity").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef union {
  double d;
  uint64_t u;
} dbits;

static double from_hilo(uint32_t hi, uint32_t lo) {
  dbits b;
  b.u = ((uint64_t)hi << 32) | lo;
  return b.d;
}
static int32_t hi_of(double x) {
  dbits b;
  b.d = x;
  return (int32_t)(b.u >> 32);
}
static uint32_t lo_of(double x) {
  dbits b;
  b.d = x;
  return (uint32_t)b.u;
}

double ox_log(double x) {
  const double ln2_hi = from_hilo(0x3fe62e42u, 0xfee00000u);
  const double ln2_lo = from_hilo(0x3dea39efu, 0x35793c76u);
  const double two54 = from_hilo(0x43500000u, 0u);
  const double Lg1 = from_hilo(0x3fe55555u, 0x55555593u);
  const double Lg2 = from_hilo(0x3fd99999u, 0x9997fa04u);
  const double Lg3 = from_hilo(0x3fd24924u, 0x94229359u);
  const double Lg4 = from_hilo(0x3fcc71c5u, 0x1d8e78afu);
  const double Lg5 = from_hilo(0x3fc74664u, 0x96cb03deu);
  const double Lg6 = from_hilo(0x3fc39a09u, 0xd078c69fu);
  const double Lg7 = from_hilo(0x3fc2f112u, 0xdf3e5244u);
  int32_t hx = hi_of(x);
  uint32_t lx = lo_of(x);
  int32_t k = 0, i, j;
  double f, s, z, w, t1, t2, R, dk, hfsq;
  if (hx < 0x00100000) {
    if (((hx & 0x7fffffff) | (int32_t)lx) == 0) return -INFINITY;
    if (hx < 0) return NAN;
    k -= 54;
    x = x * two54;
    hx = hi_of(x);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  i = (hx + 0x95f64) & 0x100000;
  x = from_hilo((uint32_t)(hx | (i ^ 0x3ff00000)), lo_of(x));
  k += (i >> 20);
  f = x - 1.0;
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      dk = (double)k;
      return dk * ln2_hi + dk * ln2_lo;
    }
    R = (f * f) * (0.5 - 0.33333333333333333 * f);
    if (k == 0) return f - R;
    dk = (double)k;
    return dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  s = f / (2.0 + f);
  dk = (double)k;
  z = s * s;
  i = hx - 0x6147a;
  w = z * z;
  j = 0x6b851 - hx;
  t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  R = t2 + t1;
  if (i > 0) {
    hfsq = (0.5 * f) * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

double ox_exp(double x) {
  const double ln2_hi = from_hilo(0x3fe62e42u, 0xfee00000u);
  const double ln2_lo = from_hilo(0x3dea39efu, 0x35793c76u);
  const double invln2 = from_hilo(0x3ff71547u, 0x652b82feu);
  const double o_thr = from_hilo(0x40862e42u, 0xfefa39efu);
  const double u_thr = from_hilo(0xc0874910u, 0xd52d3051u);
  const double twom1000 = from_hilo(0x01700000u, 0u);
  const double P1 = from_hilo(0x3fc55555u, 0x5555553eu);
  const double P2 = from_hilo(0xbf66c16cu, 0x16bebd93u);
  const double P3 = from_hilo(0x3f11566au, 0xaf25de2cu);
  const double P4 = from_hilo(0xbebbbd41u, 0xc5d26bf1u);
  const double P5 = from_hilo(0x3e663769u, 0x72bea4d0u);
  int32_t hx = hi_of(x);
  int32_t xsb = (hx >> 31) & 1;
  double hi = 0.0, lo = 0.0, t, c, y;
  int32_t k = 0;
  hx &= 0x7fffffff;
  if (hx >= 0x40862E42) {
    if (hx >= 0x7ff00000) {
      if (((hx & 0xfffff) | (int32_t)lo_of(x)) != 0) return x + x;
      return xsb == 0 ? x : 0.0;
    }
    if (x > o_thr) return INFINITY;
    if (x < u_thr) return 0.0;
  }
  if (hx > 0x3fd62e42) {
    if (hx < 0x3FF0A2B2) {
      hi = x - (xsb ? -ln2_hi : ln2_hi);
      lo = xsb ? -ln2_lo : ln2_lo;
      k = 1 - xsb - xsb;
    } else {
      k = (int32_t)(invln2 * x + (xsb ? -0.5 : 0.5));
      t = (double)k;
      hi = x - t * ln2_hi;
      lo = t * ln2_lo;
    }
    x = hi - lo;
  } else if (hx < 0x3e300000) {
    return 1.0 + x;
  } else {
    k = 0;
  }
  t = x * x;
  c = x - t * (P1 + t * (P2 + t * (P3 + t * (P4 + t * P5))));
  if (k == 0) return 1.0 - ((x * c) / (c - 2.0) - x);
  y = 1.0 - ((lo - (x * c) / (2.0 - c)) - hi);
  if (k >= -1021) return from_hilo((uint32_t)(hi_of(y) + (k << 20)), lo_of(y));
  y = from_hilo((uint32_t)(hi_of(y) + ((k + 1000) << 20)), lo_of(y));
  return y * twom1000;
}

void ox_log_array(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = ox_log(x[i]);
}
void ox_exp_array(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = ox_exp(x[i]);
}

/* canonical row sum: lane j (0..255) adds elements j, j+256, ... in order
 * starting from +0.0; lanes are then combined by a halving tree. */
double ox_canon_sum(const double* x, int64_t n) {
  double lanes[256];
  for (int j = 0; j < 256; ++j) lanes[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) lanes[i & 255] = lanes[i & 255] + x[i];
  for (int w = 128; w >= 1; w >>= 1)
    for (int j = 0; j < w; ++j) lanes[j] = lanes[j] + lanes[j + w];
  return lanes[0];
}

/* canonical inclusive scan: blocks of 256 in scan order; block totals are
 * sequential sums; the running prefix is chained block by block; inside a
 * block the scan is sequential on top of the block's incoming prefix. */
void ox_canon_cumsum(const double* x, double* out, int64_t n) {
  double prefix = 0.0;
  for (int64_t b = 0; b < n; b += 256) {
    int64_t e = b + 256 < n ? b + 256 : n;
    double local = 0.0;
    for (int64_t i = b; i < e; ++i) {
      local = local + x[i];
      out[i] = prefix + local;
    }
    prefix = prefix + local;
  }
}

/* Probability row from fp32 logits: p_v = exp(z_v - m) / S (canonical S). */
void ox_softmax_row(const float* z, int64_t V, double* p) {
  float m = z[0];
  for (int64_t v = 1; v < V; ++v)
    if (z[v] > m) m = z[v];
  for (int64_t v = 0; v < V; ++v) p[v] = ox_exp((double)z[v] - (double)m);
  double S = ox_canon_sum(p, V);
  for (int64_t v = 0; v < V; ++v) p[v] = p[v] / S;
}

/* Warp of sampling.py:66-98 under the canonical arithmetic.
 * mode 0: input are probabilities `in` (float64 row); mode 1: fp32 logits `z`.
 * temperature == 0 -> one-hot at the argmax (lowest id on ties).
 * out: warped float64 row. `order` scratch of V int32 (may be NULL if top_p==1). */
static int cmp_desc_val;
static const double* g_sort_vals;
static int cmp_pidx(const void* a, const void* b) {
  int32_t ia = *(const int32_t*)a, ib = *(const int32_t*)b;
  double va = g_sort_vals[ia], vb = g_sort_vals[ib];
  if (va > vb) return -1;
  if (va < vb) return 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

void ox_warp(const double* in_p, const float* in_z, int64_t V, double temperature, double top_p,
             double* out) {
  (void)cmp_desc_val;
  if (temperature == 0.0) {
    int64_t best = 0;
    if (in_z) {
      for (int64_t v = 1; v < V; ++v)
        if (in_z[v] > in_z[best]) best = v;
    } else {
      for (int64_t v = 1; v < V; ++v)
        if (in_p[v] > in_p[best]) best = v;
    }
    memset(out, 0, sizeof(double) * V);
    out[best] = 1.0;
    return;
  }
  if (in_z) {
    float m = in_z[0];
    for (int64_t v = 1; v < V; ++v)
      if (in_z[v] > m) m = in_z[v];
    if (temperature != 1.0) {
      double invT = 1.0 / temperature;
      for (int64_t v = 0; v < V; ++v) out[v] = ox_exp(((double)in_z[v] - (double)m) * invT);
    } else {
      for (int64_t v = 0; v < V; ++v) out[v] = ox_exp((double)in_z[v] - (double)m);
    }
    double S = ox_canon_sum(out, V);
    for (int64_t v = 0; v < V; ++v) out[v] = out[v] / S;
  } else {
    if (temperature != 1.0) {
      double invT = 1.0 / temperature;
      for (int64_t v = 0; v < V; ++v) out[v] = in_p[v] > 0.0 ? ox_exp(ox_log(in_p[v]) * invT) : 0.0;
      double S = ox_canon_sum(out, V);
      for (int64_t v = 0; v < V; ++v) out[v] = out[v] / S;
    } else {
      memcpy(out, in_p, sizeof(double) * V);
    }
  }
  if (top_p < 1.0) {
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * V);
    double* sorted = (double*)malloc(sizeof(double) * V);
    double* csum = (double*)malloc(sizeof(double) * V);
    for (int64_t v = 0; v < V; ++v) order[v] = (int32_t)v;
    g_sort_vals = out;
    qsort(order, V, sizeof(int32_t), cmp_pidx);
    for (int64_t i = 0; i < V; ++i) sorted[i] = out[order[i]];
    ox_canon_cumsum(sorted, csum, V);
    const double target = top_p - 1e-9;
    int64_t cut = V - 1;
    for (int64_t i = 0; i < V; ++i)
      if (csum[i] >= target) {
        cut = i;
        break;
      }
    /* keep order[0..cut], zero the rest, renormalise with the canonical sum */
    for (int64_t i = cut + 1; i < V; ++i) out[order[i]] = 0.0;
    double S = ox_canon_sum(out, V);
    for (int64_t v = 0; v < V; ++v) out[v] = out[v] / S;
    free(order);
    free(sorted);
    free(csum);
  }
}

/* sample (sampling.py:101-113): first index with cdf > u * cdf[-1]; fallback
 * to the largest nonzero id when it lands on a zero-probability entry. */
int64_t ox_sample(const double* p, int64_t V, double u) {
  double* cdf = (double*)malloc(sizeof(double) * V);
  ox_canon_cumsum(p, cdf, V);
  const double x = u * cdf[V - 1];
  int64_t tok = V;
  for (int64_t i = 0; i < V; ++i)
    if (cdf[i] > x) {
      tok = i;
      break;
    }
  if (tok >= V || p[tok] == 0.0) {
    tok = 0;
    for (int64_t i = V - 1; i >= 0; --i)
      if (p[i] != 0.0) {
        tok = i;
        break;
      }
  }
  free(cdf);
  return tok;
}
