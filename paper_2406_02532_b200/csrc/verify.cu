// KV1/KV2: stage-4 verification on the GPU -- the acceptance walk of
// generate_specexec (pkg/src/speckit/engine.py:118-128) over the cached target
// rows: per step sample(apply_warp(row[cursor]), u) (sampling.py:66-113), move to
// the child carrying the token (ProbCache.advance engine.py:64-70 /
// DraftTree.child_with_token tree.py:132-136), stop on a miss or after
// `max_steps` tokens. Uniforms are drawn on the host from the reference-
// compatible CounterRng and uploaded (one per potential step).
//
// Also: standalone canonical warp / softmax of rows (the drop-in apply_warp and
// ProbCache row materialisation) and per-row argmax.
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"
#include "sxmath.cuh"
#include "warp_rows.cuh"

namespace sx {

struct WalkScratch {
  double* row;  // [V]
  unsigned long long *k1, *k2;
  int *i1, *i2;
};

__global__ void __launch_bounds__(kRowThreads) verify_walk_kernel(const void* rows, int row_kind, long long ld, int V,
                                                                    const int* __restrict__ parent,
                                                                    const int* __restrict__ token, int n_nodes,
                                                                    int start_cursor, const double* __restrict__ u,
                                                                    int max_steps, double temperature, double top_p,
                                                                    int* out, WalkScratch s) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  __shared__ int s_child;
  int cursor = start_cursor;
  int emitted = 0;
  int fell = 0;
  int* toks = out + 3;
  int* path = out + 3 + max_steps;
  while (emitted < max_steps) {
    const long long r = cursor + 1;
    const float* z = row_kind == SX_ROWS_LOGITS_F32 ? reinterpret_cast<const float*>(rows) + r * ld : nullptr;
    const double* p = row_kind == SX_ROWS_PROBS_F64 ? reinterpret_cast<const double*>(rows) + r * ld : nullptr;
    int tok;
    if (row_kind == SX_ROWS_ARGMAX_PACKED) {  // KV1 keys (t = 0 only): the row's argmax is in the key
      tok = 0x7fffffff - (int)(reinterpret_cast<const long long*>(rows)[r * ld] & 0x7fffffff);
    } else if (temperature == 0.0) {
      double bv = -CUDART_INF;
      int bi = 0x7fffffff;
      for (int v = threadIdx.x; v < V; v += kRowThreads) {
        const double x = z ? (double)z[v] : p[v];
        if (x > bv) {
          bv = x;
          bi = v;
        }
      }
      tok = block_argmax(sm, bv, bi);
    } else {
      warp_row(sm, z, p, V, temperature, top_p, s.row, s.k1, s.i1, s.k2, s.i2);
      tok = sample_row(sm, s.row, V, u[emitted]);
    }
    if (threadIdx.x == 0) {
      toks[emitted] = tok;
      s_child = -1;
    }
    __syncthreads();
    // child_with_token: node ids are in insertion order and sibling tokens are
    // distinct, so the match (if any) is unique.
    for (int j = threadIdx.x; j < n_nodes; j += kRowThreads)
      if (parent[j] == cursor && token[j] == tok) s_child = j;
    __syncthreads();
    const int child = s_child;
    __syncthreads();
    ++emitted;
    if (child < 0) {
      fell = 1;
      break;
    }
    cursor = child;
    if (threadIdx.x == 0) path[emitted - 1] = child + 1;
  }
  if (threadIdx.x == 0) {
    out[0] = emitted;
    out[1] = fell;
    out[2] = cursor;
  }
}

// warp each selected row into out (fp64). row_ids == nullptr: rows 0..n-1.
__global__ void __launch_bounds__(kRowThreads) warp_rows_kernel(const void* rows, int row_kind, long long ld, int V,
                                                                  const int* row_ids, double temperature,
                                                                  double top_p, double* out, long long ldo,
                                                                  unsigned long long* k1, int* i1,
                                                                  unsigned long long* k2, int* i2) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  const int i = blockIdx.x;
  const long long r = row_ids ? row_ids[i] : i;
  const float* z = row_kind == SX_ROWS_LOGITS_F32 ? reinterpret_cast<const float*>(rows) + r * ld : nullptr;
  const double* p = row_kind == SX_ROWS_PROBS_F64 ? reinterpret_cast<const double*>(rows) + r * ld : nullptr;
  const long long o = (long long)i * V;
  warp_row(sm, z, p, V, temperature, top_p, out + (long long)i * ldo, k1 + o, i1 + o, k2 + o, i2 + o);
}

// canonical probabilities of logits rows (no warp): the float64 rows a
// LanguageModel returns (models.py:43-52), materialised on demand.
__global__ void __launch_bounds__(kRowThreads) softmax_rows_kernel(const float* rows, long long ld, int V,
                                                                     const int* row_ids, double* out, long long ldo) {
  __shared__ RowSmemLite sm;
  const int i = blockIdx.x;
  const long long r = row_ids ? row_ids[i] : i;
  const float* z = rows + r * ld;
  float m;
  double S;
  row_stats(sm, z, V, 1.0, false, m, S);
  double* o = out + (long long)i * ldo;
  for (int v = threadIdx.x; v < V; v += kRowThreads) o[v] = ddiv(sx_exp(dsub((double)z[v], (double)m)), S);
}

__global__ void __launch_bounds__(kRowThreads) argmax_rows_kernel(const void* rows, int row_kind, long long ld, int V,
                                                                    int* out) {
  __shared__ RowSmemLite sm;
  const long long r = blockIdx.x;
  double bv = -CUDART_INF;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += kRowThreads) {
    const double x = row_kind == SX_ROWS_LOGITS_F32 ? (double)reinterpret_cast<const float*>(rows)[r * ld + v]
                                                    : reinterpret_cast<const double*>(rows)[r * ld + v];
    if (x > bv) {
      bv = x;
      bi = v;
    }
  }
  const int best = block_argmax(sm, bv, bi);
  if (threadIdx.x == 0) out[r] = best;
}

// KV1 for the vocab-parallel LM head at t = 0: per row the packed key of its
// best logit, orderable(logit) << 31 | (0x7fffffff - global id). One int64 MAX
// all-reduce over the vocab shards then gives every rank the global argmax with
// the lowest id among equal logits (np.argmax) -- N x 8 bytes instead of the
// all-gather of the [N, V / n] logit slices. Exact for the walk: fp32 logits that
// differ stay distinct through the canonical exp(z - M) / S in float64, so the
// logit argmax is the probability argmax.
SX_DEV unsigned long long pack_argmax(float v, int id) {
  unsigned u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // monotone in v
  return ((unsigned long long)u << 31) | (unsigned long long)(0x7fffffff - id);
}

__global__ void __launch_bounds__(kRowThreads) argmax_packed_kernel(const float* __restrict__ z, long long ld, int Vl,
                                                                     int v0, long long* out) {
  __shared__ unsigned long long red[kRowThreads / 32];
  const long long r = blockIdx.x;
  unsigned long long best = 0;
  for (int v = threadIdx.x; v < Vl; v += kRowThreads) {
    const unsigned long long k = pack_argmax(z[r * ld + v], v0 + v);
    best = k > best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long k = __shfl_xor_sync(0xffffffffu, best, o);
    best = k > best ? k : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kRowThreads / 32; ++w) best = red[w] > best ? red[w] : best;
    out[r] = (long long)best;
  }
}

__global__ void sample_rows_kernel(const double* w, long long ld, int V, const double* u, int* out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  RowSmem& sm = *reinterpret_cast<RowSmem*>(smem_raw);
  const int i = blockIdx.x;
  const int tok = sample_row(sm, w + (long long)i * ld, V, u[i]);
  if (threadIdx.x == 0) out[i] = tok;
}

static int set_rowsmem_attr(const void* fn) { return ensure_smem_attr(fn, (int)sizeof(RowSmem)); }

}  // namespace sx

using namespace sx;

extern "C" long long sx_row_scratch_bytes(int V) {
  // row fp64 + 2 x (key u64 + idx i32), 256-B aligned pieces
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  return al(8LL * V) + 2 * al(8LL * V) + 2 * al(4LL * V);
}

extern "C" int sx_verify_walk(const void* rows, int row_kind, long long ld, int V, const int* parent, const int* token,
                              int n_nodes, int start_cursor, const double* uniforms, int max_steps, double temperature,
                              double top_p, int* out, void* scratch, cudaStream_t stream) {
  if (V < 1 || max_steps < 1) return arg_error("verify_walk: V and max_steps must be >= 1");
  if (row_kind != SX_ROWS_LOGITS_F32 && row_kind != SX_ROWS_PROBS_F64 && row_kind != SX_ROWS_ARGMAX_PACKED)
    return arg_error("verify_walk: bad row kind");
  if (temperature < 0 || !(top_p > 0 && top_p <= 1)) return arg_error("verify_walk: bad warp");
  if (row_kind == SX_ROWS_ARGMAX_PACKED && temperature != 0.0)
    return arg_error("verify_walk: argmax-only rows (KV1 keys) serve t = 0 walks only");
  if (int st = set_rowsmem_attr((const void*)verify_walk_kernel)) return st;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  uint8_t* s = reinterpret_cast<uint8_t*>(scratch);
  WalkScratch ws;
  ws.row = reinterpret_cast<double*>(s);
  ws.k1 = reinterpret_cast<unsigned long long*>(s + al(8LL * V));
  ws.k2 = reinterpret_cast<unsigned long long*>(s + 2 * al(8LL * V));
  ws.i1 = reinterpret_cast<int*>(s + 3 * al(8LL * V));
  ws.i2 = reinterpret_cast<int*>(s + 3 * al(8LL * V) + al(4LL * V));
  verify_walk_kernel<<<1, kRowThreads, sizeof(RowSmem), stream>>>(rows, row_kind, ld, V, parent, token, n_nodes,
                                                                   start_cursor, uniforms, max_steps, temperature,
                                                                   top_p, out, ws);
  SX_CHECK_LAUNCH("verify_walk_kernel");
  return SX_OK;
}

extern "C" int sx_warp_rows(const void* rows, int row_kind, long long ld, int V, const int* row_ids, int n,
                            double temperature, double top_p, double* out, long long ldo, void* scratch,
                            cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (temperature < 0 || !(top_p > 0 && top_p <= 1)) return arg_error("warp_rows: bad warp");
  if (int st = set_rowsmem_attr((const void*)warp_rows_kernel)) return st;
  // scratch: n * (2 keys + 2 idx) per element
  uint8_t* s = reinterpret_cast<uint8_t*>(scratch);
  const long long e = (long long)n * V;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  unsigned long long* k1 = reinterpret_cast<unsigned long long*>(s);
  unsigned long long* k2 = reinterpret_cast<unsigned long long*>(s + al(8 * e));
  int* i1 = reinterpret_cast<int*>(s + 2 * al(8 * e));
  int* i2 = reinterpret_cast<int*>(s + 2 * al(8 * e) + al(4 * e));
  warp_rows_kernel<<<n, kRowThreads, sizeof(RowSmem), stream>>>(rows, row_kind, ld, V, row_ids, temperature, top_p,
                                                                 out, ldo, k1, i1, k2, i2);
  SX_CHECK_LAUNCH("warp_rows_kernel");
  return SX_OK;
}

extern "C" long long sx_warp_scratch_bytes(int n, int V) {
  const long long e = (long long)n * V;
  auto al = [](long long x) { return (x + 255) & ~255LL; };
  return 2 * al(8 * e) + 2 * al(4 * e);
}

extern "C" int sx_softmax_rows(const float* rows, long long ld, int V, const int* row_ids, int n, double* out,
                               long long ldo, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  softmax_rows_kernel<<<n, kRowThreads, 0, stream>>>(rows, ld, V, row_ids, out, ldo);
  SX_CHECK_LAUNCH("softmax_rows_kernel");
  return SX_OK;
}

extern "C" int sx_argmax_rows(const void* rows, int row_kind, long long ld, int V, int n, int* out,
                              cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  argmax_rows_kernel<<<n, kRowThreads, 0, stream>>>(rows, row_kind, ld, V, out);
  SX_CHECK_LAUNCH("argmax_rows_kernel");
  return SX_OK;
}

extern "C" int sx_rows_argmax_packed(const float* logits, long long ld, int n, int Vl, int v0, long long* out,
                                     cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (Vl < 1 || v0 < 0 || ld < Vl || (long long)v0 + Vl > 0x7fffffffLL)
    return arg_error("rows_argmax_packed: bad slice (Vl=%d v0=%d ld=%lld)", Vl, v0, ld);
  argmax_packed_kernel<<<n, kRowThreads, 0, stream>>>(logits, ld, Vl, v0, out);
  SX_CHECK_LAUNCH("argmax_packed_kernel");
  return SX_OK;
}

extern "C" int sx_sample_rows(const double* w, long long ld, int V, const double* u, int n, int* out,
                              cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (int st = set_rowsmem_attr((const void*)sample_rows_kernel)) return st;
  sample_rows_kernel<<<n, kRowThreads, sizeof(RowSmem), stream>>>(w, ld, V, u, out);
  SX_CHECK_LAUNCH("sample_rows_kernel");
  return SX_OK;
}
