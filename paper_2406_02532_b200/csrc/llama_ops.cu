// KE / KV3: the HBM-bound glue of the Llama-shaped forward used by the draft
// (per tree round) and the target (one pass over the flattened tree):
//   embed        x[t]  = float(E[token[t]])                         (fp32 residual stream)
//   rmsnorm      y[t]  = bf16(x[t] * rsqrt(mean(x[t]^2) + eps) * w)
//   rope_kv      rotate q/k (rotate-half convention, per-token position
//                = len(anchor) - 1 + depth) and scatter K/V into the cache slots
//   kv_compact   move the KV rows of the accepted path [root, accepted nodes...]
//                to the committed region (no reference counterpart: the reference
//                model API is stateless, pkg/src/speckit/models.py:43-52)
// KV cache layout per layer: [KVH][slots][128] bf16 for K and for V.
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"

namespace sx {

__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, const int* __restrict__ tokens, int n, int d,
                             float* __restrict__ x) {
  griddep_launch_dependents();
  const int t = blockIdx.x;
  if (t >= n) return;
  const long long tok = tokens[t];
  const __nv_bfloat162* src = reinterpret_cast<const __nv_bfloat162*>(E + tok * d);
  float2* dst = reinterpret_cast<float2*>(x + (long long)t * d);
  for (int i = threadIdx.x; i < d / 2; i += blockDim.x) dst[i] = __bfloat1622float2(src[i]);
}

__global__ void rmsnorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w, int d, float eps,
                               __nv_bfloat16* __restrict__ y) {
  griddep_launch_dependents();
  const int t = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (long long)t * d);
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)d + eps);
  __nv_bfloat162* yr = reinterpret_cast<__nv_bfloat162*>(y + (long long)t * d);
  const __nv_bfloat162* wr = reinterpret_cast<const __nv_bfloat162*>(w);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    const float2 w0 = __bfloat1622float2(wr[2 * i]);
    const float2 w1 = __bfloat1622float2(wr[2 * i + 1]);
    yr[2 * i] = __floats2bfloat162_rn(v.x * r * w0.x, v.y * r * w0.y);
    yr[2 * i + 1] = __floats2bfloat162_rn(v.z * r * w1.x, v.w * r * w1.y);
  }
}

// Residual add fused into the following norm: x[t] += y[t] (fp32, or bf16 -- a
// tensor-parallel all-reduce result), then y_norm = bf16(rmsnorm(x[t]) * w); w
// NULL: the add only. Keeps the GEMM epilogues store-only (a cold fp32
// read-modify-write of the residual in the epilogue measured 2x on the o-proj).
template <typename T>
SX_DEV float4 ld4(const T* p, int i);
template <>
SX_DEV float4 ld4<float>(const float* p, int i) {
  return reinterpret_cast<const float4*>(p)[i];
}
template <>
SX_DEV float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p, int i) {
  const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(p);
  const float2 a = __bfloat1622float2(q[2 * i]), b = __bfloat1622float2(q[2 * i + 1]);
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename T>
__global__ void add_rmsnorm_kernel(float* __restrict__ x, const T* __restrict__ yin, const __nv_bfloat16* __restrict__ w,
                                   int d, float eps, __nv_bfloat16* __restrict__ out) {
  griddep_launch_dependents();
  const int t = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + (long long)t * d);
  const T* yr = yin + (long long)t * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    float4 v = xr[i];
    const float4 a = ld4<T>(yr, i);
    v.x += a.x;
    v.y += a.y;
    v.z += a.z;
    v.w += a.w;
    xr[i] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (w == nullptr) return;
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)d + eps);
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(out + (long long)t * d);
  const __nv_bfloat162* wr = reinterpret_cast<const __nv_bfloat162*>(w);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];  // this thread's own store above
    const float2 w0 = __bfloat1622float2(wr[2 * i]);
    const float2 w1 = __bfloat1622float2(wr[2 * i + 1]);
    o2[2 * i] = __floats2bfloat162_rn(v.x * r * w0.x, v.y * r * w0.y);
    o2[2 * i + 1] = __floats2bfloat162_rn(v.z * r * w1.x, v.w * r * w1.y);
  }
}

// qkv [n, (H + 2*KVH) * 128] bf16 -> q [n, H, 128] (rotated), K/V cache rows at slot[t].
// cos/sin tables [max_pos, 64] fp32.
__global__ void rope_kv_kernel(const __nv_bfloat16* __restrict__ qkv, const int* __restrict__ pos, int pos_base,
                               const int* __restrict__ slot, int slot_base, int n, int H, int KVH,
                               const float* __restrict__ cos_t,
                               const float* __restrict__ sin_t, __nv_bfloat16* __restrict__ q,
                               __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, long long slots) {
  const int t = blockIdx.x;
  const int heads = H + 2 * KVH;
  const int p = pos_base + (pos ? pos[t] : t);
  const long long s = slot_base + (slot ? slot[t] : t);
  const __nv_bfloat16* row = qkv + (long long)t * heads * 128;
  // one warp per head, each lane handles dims (lane, lane+32) and their +64 partners
  for (int h = threadIdx.x >> 5; h < heads; h += blockDim.x >> 5) {
    const int lane = threadIdx.x & 31;
    const __nv_bfloat16* src = row + h * 128;
    if (h < H + KVH) {
      __nv_bfloat16* dst = h < H ? q + ((long long)t * H + h) * 128 : kc + ((long long)(h - H) * slots + s) * 128;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int d = lane + 32 * k;  // 0..63
        const float c = cos_t[(long long)p * 64 + d], sn = sin_t[(long long)p * 64 + d];
        const float x0 = __bfloat162float(src[d]), x1 = __bfloat162float(src[d + 64]);
        dst[d] = __float2bfloat16(x0 * c - x1 * sn);
        dst[d + 64] = __float2bfloat16(x1 * c + x0 * sn);
      }
    } else {
      __nv_bfloat16* dst = vc + ((long long)(h - H - KVH) * slots + s) * 128;
      reinterpret_cast<uint2*>(dst)[lane] = reinterpret_cast<const uint2*>(src)[lane];
    }
  }
}

// Move KV rows src_slot[i] -> dst_slot[i] for all layers / kv heads. Rows are
// staged in shared memory first, so overlapping source/destination ranges are
// safe. A row is 128 elements: row_u4 = 16 uint4 (bf16) or 32 (fp32 mode).
__global__ void kv_compact_kernel(uint8_t* kc, uint8_t* vc, long long layer_stride_bytes, long long slots, int KVH,
                                  int row_u4, const int* __restrict__ src, const int* __restrict__ dst, int n) {
  extern __shared__ __align__(16) uint4 stage[];  // [2][n][row_u4]
  const int layer = blockIdx.y, h = blockIdx.x;
  const long long row_bytes = (long long)row_u4 * 16;
  uint8_t* kb = kc + layer * layer_stride_bytes + (long long)h * slots * row_bytes;
  uint8_t* vb = vc + layer * layer_stride_bytes + (long long)h * slots * row_bytes;
  const int total = n * row_u4;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int r = i / row_u4, c = i - r * row_u4;
    stage[i] = reinterpret_cast<const uint4*>(kb + src[r] * row_bytes)[c];
    stage[total + i] = reinterpret_cast<const uint4*>(vb + src[r] * row_bytes)[c];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int r = i / row_u4, c = i - r * row_u4;
    reinterpret_cast<uint4*>(kb + dst[r] * row_bytes)[c] = stage[i];
    reinterpret_cast<uint4*>(vb + dst[r] * row_bytes)[c] = stage[total + i];
  }
}

static int kv_compact_launch(void* kcache, void* vcache, int layers, long long layer_stride_elems, long long slots,
                             int KVH, int elem_bytes, const int* src, const int* dst, int n, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  const int row_u4 = 128 * elem_bytes / 16;
  // all rows are staged in smem (K and V of one head): up to 448 bf16 rows / 224
  // fp32 rows -- more than the deepest accepted path (max_depth <= 250 -> 251
  // rows) in bf16; fp32 mode validates its depth up front
  const int max_rows = (int)((227LL * 1024) / (2LL * row_u4 * 16));
  if (n > max_rows) return arg_error("kv_compact: at most %d rows per call (got %d)", max_rows, n);
  const size_t smem = (size_t)2 * n * row_u4 * sizeof(uint4);
  if (smem > 48 * 1024)
    if (int st = ensure_smem_attr((const void*)kv_compact_kernel, (int)smem)) return st;
  kv_compact_kernel<<<dim3(KVH, layers), 256, smem, stream>>>(reinterpret_cast<uint8_t*>(kcache),
                                                               reinterpret_cast<uint8_t*>(vcache),
                                                               layer_stride_elems * elem_bytes, slots, KVH, row_u4,
                                                               src, dst, n);
  SX_CHECK_LAUNCH("kv_compact_kernel");
  return SX_OK;
}

}  // namespace sx

using namespace sx;

extern "C" int sx_embed(const void* E, const int* tokens, int n, int d, float* x, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (d % 2) return arg_error("embed: d must be even");
  embed_kernel<<<n, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(E), tokens, n, d, x);
  SX_CHECK_LAUNCH("embed_kernel");
  return SX_OK;
}

extern "C" int sx_rmsnorm(const float* x, const void* w, int n, int d, float eps, void* y, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (d % 4) return arg_error("rmsnorm: d must be a multiple of 4");
  rmsnorm_kernel<<<n, 256, 0, stream>>>(x, reinterpret_cast<const __nv_bfloat16*>(w), d, eps,
                                        reinterpret_cast<__nv_bfloat16*>(y));
  SX_CHECK_LAUNCH("rmsnorm_kernel");
  return SX_OK;
}

// Owner-side half of the fused all-reduce (sx_gemm_bf16_rs): y_slice[t][c] =
// sum over source ranks r (in order) of inbox[r][t][c], written to every rank's
// y at columns rank * S + c (peer stores over NVLink; y fp32 or bf16).
__global__ void tp_reduce_bcast_kernel(const __nv_bfloat16* __restrict__ inbox, int rank, int world, int M, int S, int N,
                                       void* const* __restrict__ peer_y, int y_bf16) {
  const long long n = (long long)M * S / 2;  // bf16 pairs
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    for (int r = 0; r < world; ++r) {
      const float2 v = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(inbox + (long long)r * M * S)[i]);
      acc.x += v.x;
      acc.y += v.y;
    }
    const long long e = 2 * i;
    const long long t = e / S, c = e % S;
    const long long off = t * N + (long long)rank * S + c;
    for (int q = 0; q < world; ++q) {
      if (y_bf16)
        *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(peer_y[q]) + off) =
            __floats2bfloat162_rn(acc.x, acc.y);
      else
        *reinterpret_cast<float2*>(reinterpret_cast<float*>(peer_y[q]) + off) = acc;
    }
  }
}

extern "C" int sx_tp_reduce_bcast(const void* inbox, int rank, int world, int M, int N, void* const* peer_y, int y_bf16,
                                  cudaStream_t stream) {
  if (M <= 0) return SX_OK;
  if (world < 1 || rank < 0 || rank >= world || N % world || (N / world) % 2)
    return arg_error("tp_reduce_bcast: bad rank %d / world %d / N %d", rank, world, N);
  const int S = N / world;
  const long long pairs = (long long)M * S / 2;
  int grid = (int)((pairs + 255) / 256);
  if (grid > 4 * kNumSMs) grid = 4 * kNumSMs;
  tp_reduce_bcast_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(inbox), rank, world, M, S, N,
                                                   peer_y, y_bf16);
  SX_CHECK_LAUNCH("tp_reduce_bcast_kernel");
  return SX_OK;
}

extern "C" int sx_add_rmsnorm(float* x, const void* y, int y_bf16, const void* w, int n, int d, float eps, void* out,
                              cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (d % 4) return arg_error("add_rmsnorm: d must be a multiple of 4");
  if (w != nullptr && out == nullptr) return arg_error("add_rmsnorm: out is NULL");
  const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(w);
  __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(out);
  if (y_bf16)
    add_rmsnorm_kernel<__nv_bfloat16><<<n, 256, 0, stream>>>(x, reinterpret_cast<const __nv_bfloat16*>(y), wb, d, eps, ob);
  else
    add_rmsnorm_kernel<float><<<n, 256, 0, stream>>>(x, reinterpret_cast<const float*>(y), wb, d, eps, ob);
  SX_CHECK_LAUNCH("add_rmsnorm_kernel");
  return SX_OK;
}

extern "C" int sx_rope_kv(const void* qkv, const int* pos, int pos_base, const int* slot, int slot_base, int n, int H,
                          int KVH, const float* cos_t, const float* sin_t, void* q, void* kcache, void* vcache,
                          long long slots, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  rope_kv_kernel<<<n, 512, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), pos, pos_base, slot, slot_base,
                                        n, H, KVH, cos_t,
                                        sin_t, reinterpret_cast<__nv_bfloat16*>(q),
                                        reinterpret_cast<__nv_bfloat16*>(kcache),
                                        reinterpret_cast<__nv_bfloat16*>(vcache), slots);
  SX_CHECK_LAUNCH("rope_kv_kernel");
  return SX_OK;
}

extern "C" int sx_kv_compact(void* kcache, void* vcache, int layers, long long layer_stride, long long slots, int KVH,
                             const int* src, const int* dst, int n, cudaStream_t stream) {
  return kv_compact_launch(kcache, vcache, layers, layer_stride, slots, KVH, 2, src, dst, n, stream);
}

extern "C" int sx_kv_compact_f32(void* kcache, void* vcache, int layers, long long layer_stride, long long slots,
                                 int KVH, const int* src, const int* dst, int n, cudaStream_t stream) {
  return kv_compact_launch(kcache, vcache, layers, layer_stride, slots, KVH, 4, src, dst, n, stream);
}
