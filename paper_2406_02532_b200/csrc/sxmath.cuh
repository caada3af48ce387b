// Deterministic float64 log / exp for the tree-scoring and verification kernels.
//
// The reference scores every draft candidate with float64 `np.log(p)`
// (pkg/src/speckit/tree.py:230-232, :302-306) and builds probabilities with
// float64 arithmetic (pkg/src/speckit/sampling.py:66-98). CUDA's libdevice
// `log`/`exp` are not specified bit-for-bit, so the tree topology could drift on
// near-ties between runs of different toolchains. These kernels instead use a
// fixed, documented algorithm (the classic fdlibm `__ieee754_log` /
// `__ieee754_exp` reductions, < 1 ulp) evaluated with non-contracted IEEE
// double operations (__dadd_rn/__dmul_rn/...). The CPU oracle (oracle/oxmath.c)
// evaluates the same expression trees, so GPU and oracle keys agree bit-for-bit.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace sx {

#define SXM __device__ __forceinline__
SXM double dadd(double a, double b) { return __dadd_rn(a, b); }
SXM double dsub(double a, double b) { return __dsub_rn(a, b); }
SXM double dmul(double a, double b) { return __dmul_rn(a, b); }
SXM double ddiv(double a, double b) { return __ddiv_rn(a, b); }

SXM double hex2d(unsigned hi, unsigned lo) { return __hiloint2double((int)hi, (int)lo); }

SXM double sx_log(double x) {
  const double ln2_hi = hex2d(0x3fe62e42u, 0xfee00000u);
  const double ln2_lo = hex2d(0x3dea39efu, 0x35793c76u);
  const double two54 = hex2d(0x43500000u, 0u);
  const double Lg1 = hex2d(0x3fe55555u, 0x55555593u);
  const double Lg2 = hex2d(0x3fd99999u, 0x9997fa04u);
  const double Lg3 = hex2d(0x3fd24924u, 0x94229359u);
  const double Lg4 = hex2d(0x3fcc71c5u, 0x1d8e78afu);
  const double Lg5 = hex2d(0x3fc74664u, 0x96cb03deu);
  const double Lg6 = hex2d(0x3fc39a09u, 0xd078c69fu);
  const double Lg7 = hex2d(0x3fc2f112u, 0xdf3e5244u);

  int hx = __double2hiint(x);
  unsigned lx = (unsigned)__double2loint(x);
  int k = 0;
  if (hx < 0x00100000) {
    if (((hx & 0x7fffffff) | (int)lx) == 0) return -CUDART_INF;
    if (hx < 0) return CUDART_NAN;
    k -= 54;
    x = dmul(x, two54);
    hx = __double2hiint(x);
  }
  if (hx >= 0x7ff00000) return dadd(x, x);
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int i = (hx + 0x95f64) & 0x100000;
  x = __hiloint2double(hx | (i ^ 0x3ff00000), __double2loint(x));
  k += (i >> 20);
  const double f = dsub(x, 1.0);
  double dk, R;
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      dk = (double)k;
      return dadd(dmul(dk, ln2_hi), dmul(dk, ln2_lo));
    }
    R = dmul(dmul(f, f), dsub(0.5, dmul(0.33333333333333333, f)));
    if (k == 0) return dsub(f, R);
    dk = (double)k;
    return dsub(dmul(dk, ln2_hi), dsub(dsub(R, dmul(dk, ln2_lo)), f));
  }
  const double s = ddiv(f, dadd(2.0, f));
  dk = (double)k;
  const double z = dmul(s, s);
  i = hx - 0x6147a;
  const double w = dmul(z, z);
  const int j = 0x6b851 - hx;
  const double t1 = dmul(w, dadd(Lg2, dmul(w, dadd(Lg4, dmul(w, Lg6)))));
  const double t2 = dmul(z, dadd(Lg1, dmul(w, dadd(Lg3, dmul(w, dadd(Lg5, dmul(w, Lg7)))))));
  i |= j;
  R = dadd(t2, t1);
  if (i > 0) {
    const double hfsq = dmul(dmul(0.5, f), f);
    if (k == 0) return dsub(f, dsub(hfsq, dmul(s, dadd(hfsq, R))));
    return dsub(dmul(dk, ln2_hi), dsub(dsub(hfsq, dadd(dmul(s, dadd(hfsq, R)), dmul(dk, ln2_lo))), f));
  }
  if (k == 0) return dsub(f, dmul(s, dsub(f, R)));
  return dsub(dmul(dk, ln2_hi), dsub(dsub(dmul(s, dsub(f, R)), dmul(dk, ln2_lo)), f));
}

SXM double sx_exp(double x) {
  const double ln2_hi = hex2d(0x3fe62e42u, 0xfee00000u);
  const double ln2_lo = hex2d(0x3dea39efu, 0x35793c76u);
  const double invln2 = hex2d(0x3ff71547u, 0x652b82feu);
  const double o_thr = hex2d(0x40862e42u, 0xfefa39efu);
  const double u_thr = hex2d(0xc0874910u, 0xd52d3051u);
  const double twom1000 = hex2d(0x01700000u, 0u);
  const double P1 = hex2d(0x3fc55555u, 0x5555553eu);
  const double P2 = hex2d(0xbf66c16cu, 0x16bebd93u);
  const double P3 = hex2d(0x3f11566au, 0xaf25de2cu);
  const double P4 = hex2d(0xbebbbd41u, 0xc5d26bf1u);
  const double P5 = hex2d(0x3e663769u, 0x72bea4d0u);

  int hx = __double2hiint(x);
  const int xsb = (hx >> 31) & 1;
  hx &= 0x7fffffff;
  if (hx >= 0x40862E42) {
    if (hx >= 0x7ff00000) {
      if (((hx & 0xfffff) | __double2loint(x)) != 0) return dadd(x, x);
      return xsb == 0 ? x : 0.0;
    }
    if (x > o_thr) return CUDART_INF;
    if (x < u_thr) return 0.0;
  }
  double hi = 0.0, lo = 0.0;
  int k = 0;
  if (hx > 0x3fd62e42) {
    if (hx < 0x3FF0A2B2) {
      hi = dsub(x, xsb ? -ln2_hi : ln2_hi);
      lo = xsb ? -ln2_lo : ln2_lo;
      k = 1 - xsb - xsb;
    } else {
      k = __double2int_rz(dadd(dmul(invln2, x), xsb ? -0.5 : 0.5));
      const double t = (double)k;
      hi = dsub(x, dmul(t, ln2_hi));
      lo = dmul(t, ln2_lo);
    }
    x = dsub(hi, lo);
  } else if (hx < 0x3e300000) {
    return dadd(1.0, x);
  } else {
    k = 0;
  }
  const double t = dmul(x, x);
  const double c =
      dsub(x, dmul(t, dadd(P1, dmul(t, dadd(P2, dmul(t, dadd(P3, dmul(t, dadd(P4, dmul(t, P5))))))))));
  if (k == 0) return dsub(1.0, dsub(ddiv(dmul(x, c), dsub(c, 2.0)), x));
  double y = dsub(1.0, dsub(dsub(lo, ddiv(dmul(x, c), dsub(2.0, c))), hi));
  if (k >= -1021) {
    return __hiloint2double(__double2hiint(y) + (k << 20), __double2loint(y));
  }
  y = __hiloint2double(__double2hiint(y) + ((k + 1000) << 20), __double2loint(y));
  return dmul(y, twom1000);
}

#undef SXM
}  // namespace sx
