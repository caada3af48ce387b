// SpecInfer baseline on the GPU: the stochastic draft
// tree's sampling step and the multi-round rejection verification walk of
// pkg/src/speckit/specinfer.py:53-96 / tree.py:383-425, with the same canonical
// float64 arithmetic as the SpecExec kernels (warp_rows.cuh) and as the CPU
// oracle (oracle/speckit_oracle.py build_stochastic / verify_specinfer).
//
//   KI1 sample_rows_idx : token = sample(q[row_ids[i]], u[i]) plus its edge
//                         log q[token] (tree.py:415-419) -- the `width` i.i.d.
//                         draws per expanded node of one level, in one launch
//   KI2 specinfer_verify: one CTA walks the tree: p = warp(target row of the
//                         node); for each child in id order, `multiplicity`
//                         trials u < min(1, p[x] / q[x]); a rejection moves p to
//                         normalize(max(p - q, 0)) (specinfer.py:42-50); no
//                         acceptance -> bonus = sample(p, u). Uniforms are the
//                         host CounterRng "specinfer-accept" stream, pre-drawn
//                         (an upper bound); the kernel reports how many it used.
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"
#include "sxmath.cuh"
#include "warp_rows.cuh"

namespace sx {

__global__ void __launch_bounds__(kRowThreads) sample_rows_idx_kernel(const double* w, long long ld, int V,
                                                                        const int* row_ids, const double* u,
                                                                        int* out_tok, double* out_logq) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  const int i = blockIdx.x;
  const double* row = w + (long long)(row_ids ? row_ids[i] : i) * ld;
  const int tok = sample_row(sm, row, V, u[i]);
  if (threadIdx.x == 0) {
    out_tok[i] = tok;
    if (out_logq) out_logq[i] = sx_log(row[tok]);
  }
}

struct SiScratch {
  double* p;  // [V] current target distribution (warped, then residuals)
  unsigned long long *k1, *k2;
  int *i1, *i2;
};

// p <- normalize(max(p - q, 0)) unless the mass is zero; returns 1 when the
// result fails validate_distribution (|sum - 1| > 1e-9), 0 otherwise.
SX_DEV int residual_inplace(RowSmem& sm, double* p, const double* q, int V) {
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int v = t; v < V; v += kRowThreads) acc = dadd(acc, fmax(dsub(p[v], q[v]), 0.0));
  const double total = block_canon_sum(sm, acc);
  if (!(total > 0.0)) return 0;  // specinfer.py:45-49: residual undefined -> keep p
  double acc2 = 0.0;
  for (int v = t; v < V; v += kRowThreads) {
    const double r = ddiv(fmax(dsub(p[v], q[v]), 0.0), total);
    p[v] = r;
    acc2 = dadd(acc2, r);
  }
  const double s = block_canon_sum(sm, acc2);  // also orders the stores above
  return fabs(dsub(s, 1.0)) > 1e-9 ? 1 : 0;
}

// Tree rows: row 0 = root (anchor), row n+1 = node n. Per row r: children are
// the node ids [child_start[r], child_start[r] + child_count[r]) (a stochastic
// tree assigns ids level by level, a node's samples consecutively), q_row[r] =
// index of the distribution its children were drawn from (-1: not expanded).
__global__ void __launch_bounds__(kRowThreads) specinfer_verify_kernel(
    const void* trows, int row_kind, long long ld, int V, const double* __restrict__ q, long long ldq,
    const int* __restrict__ q_row, const int* __restrict__ child_start, const int* __restrict__ child_count,
    const int* __restrict__ token, const int* __restrict__ mult, int max_path, const double* __restrict__ u, int n_u,
    double temperature, double top_p, int* out, SiScratch s) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  int node = -1, plen = 0, k = 0, err = 0, bonus = -1;
  auto row_z = [&](int r) -> const float* {
    return row_kind == SX_ROWS_LOGITS_F32 ? reinterpret_cast<const float*>(trows) + (long long)r * ld : nullptr;
  };
  auto row_p = [&](int r) -> const double* {
    return row_kind == SX_ROWS_PROBS_F64 ? reinterpret_cast<const double*>(trows) + (long long)r * ld : nullptr;
  };
  warp_row(sm, row_z(0), row_p(0), V, temperature, top_p, s.p, s.k1, s.i1, s.k2, s.i2);
  while (true) {
    const int r = node + 1;
    const int c0 = child_start[r], cn = child_count[r], qi = q_row[r];
    int accepted = -1;
    if (cn > 0 && qi < 0) {
      err = 2;  // children without the distribution they were drawn from
      break;
    }
    for (int c = c0; c < c0 + cn && accepted < 0 && !err; ++c) {
      const double* qr = q + (long long)qi * ldq;
      const int tok = token[c];
      for (int j = 0; j < mult[c]; ++j) {
        if (k >= n_u) {
          err = 3;  // ran out of pre-drawn uniforms
          break;
        }
        const double ratio = fmin(1.0, ddiv(s.p[tok], qr[tok]));
        const double uu = u[k++];
        if (uu < ratio) {
          accepted = c;
          break;
        }
        if (residual_inplace(sm, s.p, qr, V)) {
          err = 1;  // validate_distribution would raise (sampling.py:44-56)
          break;
        }
      }
    }
    if (err) break;
    if (accepted < 0) {
      if (k >= n_u) {
        err = 3;
        break;
      }
      bonus = sample_row(sm, s.p, V, u[k++]);
      break;
    }
    if (threadIdx.x == 0 && plen < max_path) out[4 + plen] = accepted;
    ++plen;
    node = accepted;
    __syncthreads();
    warp_row(sm, row_z(node + 1), row_p(node + 1), V, temperature, top_p, s.p, s.k1, s.i1, s.k2, s.i2);
  }
  if (threadIdx.x == 0) {
    out[0] = plen;
    out[1] = bonus;
    out[2] = k;
    out[3] = err;
  }
}

}  // namespace sx

using namespace sx;

extern "C" int sx_sample_rows_idx(const double* w, long long ld, int V, const int* row_ids, const double* u, int n,
                                  int* out_tok, double* out_logq, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (V < 1) return arg_error("sample_rows_idx: V must be >= 1");
  if (int st = ensure_smem_attr((const void*)sample_rows_idx_kernel, (int)sizeof(RowSmem))) return st;
  sample_rows_idx_kernel<<<n, kRowThreads, sizeof(RowSmem), stream>>>(w, ld, V, row_ids, u, out_tok, out_logq);
  SX_CHECK_LAUNCH("sample_rows_idx_kernel");
  return SX_OK;
}

extern "C" int sx_specinfer_verify(const void* trows, int row_kind, long long ld, int V, const double* q,
                                   long long ldq, const int* q_row, const int* child_start, const int* child_count,
                                   const int* token, const int* mult, int max_path, const double* uniforms, int n_u,
                                   double temperature, double top_p, int* out, void* scratch, cudaStream_t stream) {
  if (V < 1 || max_path < 0) return arg_error("specinfer_verify: V must be >= 1, max_path >= 0");
  if (row_kind != SX_ROWS_LOGITS_F32 && row_kind != SX_ROWS_PROBS_F64)
    return arg_error("specinfer_verify: bad row kind");
  if (temperature < 0 || !(top_p > 0 && top_p <= 1)) return arg_error("specinfer_verify: bad warp");
  if (int st = ensure_smem_attr((const void*)specinfer_verify_kernel, (int)sizeof(RowSmem))) return st;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  uint8_t* b = reinterpret_cast<uint8_t*>(scratch);
  SiScratch s;
  s.p = reinterpret_cast<double*>(b);
  s.k1 = reinterpret_cast<unsigned long long*>(b + al(8LL * V));
  s.k2 = reinterpret_cast<unsigned long long*>(b + 2 * al(8LL * V));
  s.i1 = reinterpret_cast<int*>(b + 3 * al(8LL * V));
  s.i2 = reinterpret_cast<int*>(b + 3 * al(8LL * V) + al(4LL * V));
  specinfer_verify_kernel<<<1, kRowThreads, sizeof(RowSmem), stream>>>(
      trows, row_kind, ld, V, q, ldq, q_row, child_start, child_count, token, mult, max_path, uniforms, n_u,
      temperature, top_p, out, s);
  SX_CHECK_LAUNCH("specinfer_verify_kernel");
  return SX_OK;
}
