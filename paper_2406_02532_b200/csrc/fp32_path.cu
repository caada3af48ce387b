// fp32 target mode (north_star: "target logits within ... 1e-4 in fp32"): the
// same Llama forward as the bf16 path with every operand, activation, KV-cache
// row and accumulator in IEEE fp32 -- CUDA-core FFMA, no tensor cores (TF32 and
// bf16 splits do not carry a 24-bit mantissa through the products). It is the
// precision mode, not the throughput mode: a 2-layer 70B-width pass runs in
// milliseconds, a full 70B fp32 model does not fit one B200 (280 GB).
//
//   sx_gemm_f32          out[t, f] (op)= sum_k X[t, k] W[f, k]; epilogues: store,
//                        add, interleaved SwiGLU (gate/up in 64-row blocks, the
//                        bf16 path's "wgu" layout)
//   sx_tree_attention_f32  one warp per (token, query head): online softmax over
//                        the token's key space -- committed slots [0, dense_len)
//                        then its ancestor slots (the flattened tree mask of
//                        pkg/src/speckit/tree.py:208-219), exactly the key set of
//                        the bf16 kernels in attention.cu
//   sx_embed_f32 / sx_rmsnorm_f32 / sx_add_rmsnorm_f32 / sx_rope_kv_f32
//                        the glue of llama_ops.cu with fp32 weights and outputs
#include "capi_util.h"
#include "common.cuh"
#include "specexec_b200.h"

namespace sx {

// ---------------------------------------------------------------------------
// SIMT GEMM: 128 weight rows x 64 tokens per CTA, k-blocks of 16 staged in smem
// (transposed so each thread reads 8 weight rows and 4 tokens per k as float4s),
// 256 threads x (8 x 4) accumulators, k summed in ascending order per output
// (per k-block partial sums, then the running total).
// ---------------------------------------------------------------------------
constexpr int kFBM = 128, kFBN = 64, kFBK = 16, kFThreads = 256;

template <int EPI>
__global__ void __launch_bounds__(kFThreads) gemm_f32_kernel(const float* __restrict__ W, const float* __restrict__ X,
                                                             float* __restrict__ out, int M, int N, int K,
                                                             long long ldo) {
  __shared__ __align__(16) float As[kFBK][kFBM];
  __shared__ __align__(16) float Bs[kFBK][kFBN];
  __shared__ __align__(16) float Cs[EPI == SX_EPI_SWIGLU_IL ? kFBM : 1][kFBN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int f0 = blockIdx.x * kFBM, t0 = blockIdx.y * kFBN;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += kFBK) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {  // weight tile: 128 rows x 16 k = 512 float4
      const int idx = tid * 2 + r, row = idx >> 2, c4 = (idx & 3) * 4;
      const int f = f0 + row, k = k0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < N && k < K) v = *reinterpret_cast<const float4*>(W + (long long)f * K + k);
      As[c4 + 0][row] = v.x;
      As[c4 + 1][row] = v.y;
      As[c4 + 2][row] = v.z;
      As[c4 + 3][row] = v.w;
    }
    {  // token tile: 64 rows x 16 k = 256 float4
      const int row = tid >> 2, c4 = (tid & 3) * 4;
      const int t = t0 + row, k = k0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < M && k < K) v = *reinterpret_cast<const float4*>(X + (long long)t * K + k);
      Bs[c4 + 0][row] = v.x;
      Bs[c4 + 1][row] = v.y;
      Bs[c4 + 2][row] = v.z;
      Bs[c4 + 3][row] = v.w;
    }
    __syncthreads();
    // two-level sum: each 16-wide k-block into a fresh partial, then into the
    // running total -- rounding error grows with 16 + K/16 terms, not K
    float part[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[i][j] = 0.f;
#pragma unroll
    for (int kk = 0; kk < kFBK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) part[i][j] = fmaf(a[i], bb[j], part[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];
    __syncthreads();
  }

  if (EPI == SX_EPI_SWIGLU_IL) {
    // rows [0, 64) of the tile are gate features f0/2 + j, rows [64, 128) the up
    // projections of the same features: out[t, f0/2 + j] = silu(gate) * up
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) Cs[ty * 8 + i][tx * 4 + j] = acc[i][j];
    __syncthreads();
    for (int e = tid; e < 64 * kFBN; e += kFThreads) {
      const int j = e & 63, tl = e >> 6, t = t0 + tl;
      if (t >= M || f0 + j >= N) continue;
      const float g = Cs[j][tl], u = Cs[64 + j][tl];
      out[(long long)t * ldo + f0 / 2 + j] = g / (1.f + expf(-g)) * u;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = t0 + tx * 4 + j;
    if (t >= M) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = f0 + ty * 8 + i;
      if (f >= N) continue;
      float* o = out + (long long)t * ldo + f;
      if (EPI == SX_EPI_ADD_F32)
        *o += acc[i][j];
      else
        *o = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// attention: grid (N tokens, KVH), one warp per query head of the KV group;
// lane l holds dims [4l, 4l+4) of q / o. Keys in order: dense slots, ancestors.
// ---------------------------------------------------------------------------
__global__ void tree_attention_f32_kernel(const float* __restrict__ q, const float* __restrict__ kc,
                                          const float* __restrict__ vc, long long slots,
                                          const int* __restrict__ dense_len, int dense_const,
                                          const int* __restrict__ anc, int anc_base, const int* __restrict__ anc_len,
                                          int A, float* __restrict__ out, int H, int KVH, float scale) {
  const int t = blockIdx.x, kvh = blockIdx.y, G = H / KVH;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= G) return;
  const int h = kvh * G + w;
  const float4 qv = reinterpret_cast<const float4*>(q + ((long long)t * H + h) * 128)[lane];
  const float* kb = kc + (long long)kvh * slots * 128;
  const float* vb = vc + (long long)kvh * slots * 128;
  const int nd = dense_len ? dense_len[t] : dense_const;
  const int na = (anc && anc_len) ? anc_len[t] : 0;
  float m = -INFINITY, l = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = 0; j < nd + na; ++j) {
    const long long s = j < nd ? j : (long long)anc_base + anc[(long long)t * A + (j - nd)];
    const float4 kv = reinterpret_cast<const float4*>(kb + s * 128)[lane];
    float dot = qv.x * kv.x + qv.y * kv.y + qv.z * kv.z + qv.w * kv.w;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float sc = dot * scale;
    const float mn = fmaxf(m, sc);
    const float corr = expf(m - mn), p = expf(sc - mn);
    const float4 vv = reinterpret_cast<const float4*>(vb + s * 128)[lane];
    l = l * corr + p;
    o.x = o.x * corr + p * vv.x;
    o.y = o.y * corr + p * vv.y;
    o.z = o.z * corr + p * vv.z;
    o.w = o.w * corr + p * vv.w;
    m = mn;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  reinterpret_cast<float4*>(out + ((long long)t * H + h) * 128)[lane] =
      make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
}

// ---------------------------------------------------------------------------
// glue
// ---------------------------------------------------------------------------
__global__ void embed_f32_kernel(const float* __restrict__ E, const int* __restrict__ tokens, int d,
                                 float* __restrict__ x) {
  const int t = blockIdx.x;
  const float4* src = reinterpret_cast<const float4*>(E + (long long)tokens[t] * d);
  float4* dst = reinterpret_cast<float4*>(x + (long long)t * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = src[i];
}

SX_DEV float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// x[t] += y[t] (y may be NULL), then out[t] = x[t] * rsqrt(mean(x^2) + eps) * w (w NULL: add only)
__global__ void add_rmsnorm_f32_kernel(float* __restrict__ x, const float* __restrict__ y, const float* __restrict__ w,
                                       int d, float eps, float* __restrict__ out) {
  const int t = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + (long long)t * d);
  const float4* yr = y ? reinterpret_cast<const float4*>(y + (long long)t * d) : nullptr;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    float4 v = xr[i];
    if (yr) {
      const float4 a = yr[i];
      v.x += a.x;
      v.y += a.y;
      v.z += a.z;
      v.w += a.w;
      xr[i] = v;
    }
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (w == nullptr) return;
  __shared__ float red[32];
  const float r = rsqrtf(block_sum(ss, red) / (float)d + eps);
  const float4* wr = reinterpret_cast<const float4*>(w);
  float4* o4 = reinterpret_cast<float4*>(out + (long long)t * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i], g = wr[i];
    o4[i] = make_float4(v.x * r * g.x, v.y * r * g.y, v.z * r * g.z, v.w * r * g.w);
  }
}

// qkv [n, (H + 2 KVH) * 128] fp32 -> q [n, H, 128] rotated, K / V cache rows at the token's slot
__global__ void rope_kv_f32_kernel(const float* __restrict__ qkv, const int* __restrict__ pos, int pos_base,
                                   const int* __restrict__ slot, int slot_base, int H, int KVH,
                                   const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                   float* __restrict__ q, float* __restrict__ kc, float* __restrict__ vc,
                                   long long slots) {
  const int t = blockIdx.x, heads = H + 2 * KVH;
  const int p = pos_base + (pos ? pos[t] : t);
  const long long s = slot_base + (slot ? slot[t] : t);
  const float* row = qkv + (long long)t * heads * 128;
  for (int h = threadIdx.x >> 5; h < heads; h += blockDim.x >> 5) {
    const int lane = threadIdx.x & 31;
    const float* src = row + h * 128;
    if (h < H + KVH) {
      float* dst = h < H ? q + ((long long)t * H + h) * 128 : kc + ((long long)(h - H) * slots + s) * 128;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int d = lane + 32 * k;
        const float c = cos_t[(long long)p * 64 + d], sn = sin_t[(long long)p * 64 + d];
        const float x0 = src[d], x1 = src[d + 64];
        dst[d] = x0 * c - x1 * sn;
        dst[d + 64] = x1 * c + x0 * sn;
      }
    } else {
      float* dst = vc + ((long long)(h - H - KVH) * slots + s) * 128;
      reinterpret_cast<float4*>(dst)[lane] = reinterpret_cast<const float4*>(src)[lane];
    }
  }
}

}  // namespace sx

using namespace sx;

extern "C" int sx_gemm_f32(const float* w, const float* x, float* out, int M, int N, int K, long long ldo, int epi,
                           cudaStream_t stream) {
  if (M <= 0) return SX_OK;
  if (N <= 0 || K <= 0 || K % 4) return arg_error("gemm_f32: need N > 0 and K a positive multiple of 4 (N=%d K=%d)", N, K);
  if (((uintptr_t)w | (uintptr_t)x) & 15) return arg_error("gemm_f32: operands must be 16-byte aligned");
  dim3 grid((N + kFBM - 1) / kFBM, (M + kFBN - 1) / kFBN);
  if (grid.y > 65535) return arg_error("gemm_f32: M=%d too large", M);
  switch (epi) {
    case SX_EPI_F32:
      if (ldo < N) return arg_error("gemm_f32: ldo %lld < N %d", ldo, N);
      gemm_f32_kernel<SX_EPI_F32><<<grid, kFThreads, 0, stream>>>(w, x, out, M, N, K, ldo);
      break;
    case SX_EPI_ADD_F32:
      if (ldo < N) return arg_error("gemm_f32: ldo %lld < N %d", ldo, N);
      gemm_f32_kernel<SX_EPI_ADD_F32><<<grid, kFThreads, 0, stream>>>(w, x, out, M, N, K, ldo);
      break;
    case SX_EPI_SWIGLU_IL:
      if (N % 128) return arg_error("gemm_f32: SwiGLU needs N (%d) a multiple of 128", N);
      if (ldo < N / 2) return arg_error("gemm_f32: ldo %lld < N/2 %d", ldo, N / 2);
      gemm_f32_kernel<SX_EPI_SWIGLU_IL><<<grid, kFThreads, 0, stream>>>(w, x, out, M, N, K, ldo);
      break;
    default:
      return arg_error("gemm_f32: epilogue %d not supported (F32, ADD_F32, SWIGLU_IL)", epi);
  }
  SX_CHECK_LAUNCH("gemm_f32_kernel");
  return SX_OK;
}

extern "C" int sx_tree_attention_f32(const float* q, const float* kcache, const float* vcache, long long slots,
                                     const int* dense_len, int dense_const, const int* anc, int anc_base,
                                     const int* anc_len, int A, float* out, int N, int H, int KVH,
                                     cudaStream_t stream) {
  if (N <= 0) return SX_OK;
  if (KVH <= 0 || H % KVH || H / KVH > 32) return arg_error("attention_f32: H %d / KVH %d", H, KVH);
  if (A < 0) return arg_error("attention_f32: negative ancestor width %d", A);
  dim3 grid(N, KVH);
  tree_attention_f32_kernel<<<grid, 32 * (H / KVH), 0, stream>>>(q, kcache, vcache, slots, dense_len, dense_const, anc,
                                                                 anc_base, anc_len, A, out, H, KVH,
                                                                 1.f / sqrtf(128.f));
  SX_CHECK_LAUNCH("tree_attention_f32_kernel");
  return SX_OK;
}

extern "C" int sx_embed_f32(const float* E, const int* tokens, int n, int d, float* x, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (d % 4) return arg_error("embed_f32: d must be a multiple of 4");
  embed_f32_kernel<<<n, 256, 0, stream>>>(E, tokens, d, x);
  SX_CHECK_LAUNCH("embed_f32_kernel");
  return SX_OK;
}

extern "C" int sx_add_rmsnorm_f32(float* x, const float* y, const float* w, int n, int d, float eps, float* out,
                                  cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  if (d % 4) return arg_error("add_rmsnorm_f32: d must be a multiple of 4");
  if (w != nullptr && out == nullptr) return arg_error("add_rmsnorm_f32: out is NULL");
  add_rmsnorm_f32_kernel<<<n, 256, 0, stream>>>(x, y, w, d, eps, out);
  SX_CHECK_LAUNCH("add_rmsnorm_f32_kernel");
  return SX_OK;
}

extern "C" int sx_rope_kv_f32(const float* qkv, const int* pos, int pos_base, const int* slot, int slot_base, int n,
                              int H, int KVH, const float* cos_t, const float* sin_t, float* q, float* kcache,
                              float* vcache, long long slots, cudaStream_t stream) {
  if (n <= 0) return SX_OK;
  rope_kv_f32_kernel<<<n, 512, 0, stream>>>(qkv, pos, pos_base, slot, slot_base, H, KVH, cos_t, sin_t, q, kcache,
                                            vcache, slots);
  SX_CHECK_LAUNCH("rope_kv_f32_kernel");
  return SX_OK;
}
