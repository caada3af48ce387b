// Streaming-read probe (tools only): how fast can one kernel pull a weight matrix
// through shared memory on B200? Variants: 1-D bulk copies of S bytes (one
// producer thread, R-deep ring), 2-D tensor-map TMA boxes, plain 16-B loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2406_02532_b200/csrc stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace sx;

__global__ void __launch_bounds__(288, 1) bulk_kernel(const uint8_t* W, long long bytes, int seg, int ring, int per_stage,
                                                       float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int stage = seg * per_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ring * stage);
  uint64_t* empty = full + ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nst = bytes / stage;
  const long long s0 = nst * blockIdx.x / gridDim.x, s1 = nst * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 8);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0, ph = 0;
      for (long long i = s0; i < s1; ++i) {
        if (i - s0 >= ring) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], stage);
        for (int q = 0; q < per_stage; ++q) bulk_load(sm + s * stage + q * seg, W + i * stage + q * seg, seg, &full[s], pol);
        if (++s == ring) s = 0, ph ^= 1;
      }
    }
    return;
  }
  float acc = 0.f;
  int s = 0, ph = 0;
  for (long long i = s0; i < s1; ++i) {
    mbar_wait(&full[s], ph);
    const float4* p = reinterpret_cast<const float4*>(sm + s * stage);
    for (int v = threadIdx.x; v < stage / 16; v += 256) acc += p[v].x;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == ring) s = 0, ph ^= 1;
  }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(288, 1) tmap_kernel(const __grid_constant__ CUtensorMap map, int rows, int cols,
                                                       int boxr, int boxc, int ring, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int stage = boxr * boxc * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ring * stage);
  uint64_t* empty = full + ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nr = rows / boxr, nc = cols / boxc, nst = nr * nc;
  const long long s0 = nst * blockIdx.x / gridDim.x, s1 = nst * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 8);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      int s = 0, ph = 0;
      for (long long i = s0; i < s1; ++i) {
        if (i - s0 >= ring) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], stage);
        tma_load_2d(sm + s * stage, &map, &full[s], (int)(i % nc) * boxc, (int)(i / nc) * boxr);
        if (++s == ring) s = 0, ph ^= 1;
      }
    }
    return;
  }
  float acc = 0.f;
  int s = 0, ph = 0;
  for (long long i = s0; i < s1; ++i) {
    mbar_wait(&full[s], ph);
    const float4* p = reinterpret_cast<const float4*>(sm + s * stage);
    for (int v = threadIdx.x; v < stage / 16; v += 256) acc += p[v].x;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == ring) s = 0, ph ^= 1;
  }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void ldg_kernel(const uint4* W, long long n16, float* sink) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __ldcs(W + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += __int_as_float(a[k].x);
  }
  for (; i < n16; i += stride) acc += __int_as_float(__ldcs(W + i).x);
  if (acc == 12345.f) sink[0] = acc;
}


// gemv pattern: stage = R row segments of KC columns (row stride K), rows either
// consecutive or in (f, f+64) pairs; a CTA walks its contiguous range of row groups
__global__ void __launch_bounds__(288, 1) rows_kernel(const uint8_t* W, int N, int K, int R, int KC, int ring, int paired,
                                                       float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int stage = R * KC * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ring * stage);
  uint64_t* empty = full + ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = N / R, nchunk = K / KC;
  const long long g0 = (long long)groups * blockIdx.x / gridDim.x, g1 = (long long)groups * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 8);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0, ph = 0, n = 0;
      for (long long gi = g0; gi < g1; ++gi)
        for (int c = 0; c < nchunk; ++c, ++n) {
          if (n >= ring) mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], stage);
          for (int q = 0; q < R; ++q) {
            long long row;
            if (paired) {  // group gi = 8 pairs of tile gi / 8 ... (pairs p = gi*R/2 + q/2)
              const long long p = gi * (R / 2) + (q >> 1);
              row = (p >> 6) * 128 + (p & 63) + (q & 1) * 64;
            } else {
              row = gi * R + q;
            }
            bulk_load(sm + s * stage + q * KC * 2, W + row * K * 2 + (long long)c * KC * 2, KC * 2, &full[s], pol);
          }
          if (++s == ring) s = 0, ph ^= 1;
        }
    }
    return;
  }
  float acc = 0.f;
  int s = 0, ph = 0;
  for (long long gi = g0; gi < g1; ++gi)
    for (int c = 0; c < nchunk; ++c) {
      mbar_wait(&full[s], ph);
      const float4* p = reinterpret_cast<const float4*>(sm + s * stage);
      for (int v = threadIdx.x; v < stage / 16; v += 256) acc += p[v].x;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == ring) s = 0, ph ^= 1;
    }
  if (acc == 12345.f) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const long long bytes = argc > 1 ? atoll(argv[1]) : 180LL << 20;
  uint8_t* W;
  float* sink;
  cudaMalloc(&W, bytes + (1 << 20));
  cudaMalloc(&sink, 4);
  cudaMemset(W, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    return ms / it * 1e3;
  };
  if (argc > 3) {
  cudaFuncSetAttribute(rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  {
    const int K = argc > 2 ? atoi(argv[2]) : 4096;
    const int N = (int)(bytes / (K * 2)) / 128 * 128;
    for (int paired : {0, 1})
      for (int R : {4, 8, 16})
        for (int KC : {512, 1024, 2048, 4096})
          for (int ringkb : {64, 128, 192}) {
            const int stage = R * KC * 2;
            const int ring = ringkb * 1024 / stage;
            if (ring < 2 || KC > K || ring * stage + 16 * ring + 64 > 227 * 1024) continue;
            const float us = timeit([&] { rows_kernel<<<148, 288, ring * stage + 16 * ring + 64>>>(W, N, K, R, KC, ring, paired, sink); });
            printf("{\"kind\": \"rows\", \"K\": %d, \"paired\": %d, \"R\": %d, \"KC\": %d, \"ring\": %d, \"us\": %.1f, \"GBps\": %.0f}\n",
                   K, paired, R, KC, ring, us, (double)N * K * 2 / us / 1e3);
          }
  }
  return 0;
  }
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(tmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int segs[] = {1024, 2048, 4096, 8192, 16384};
  for (int seg : segs)
    for (int per : {1, 4, 16})
      for (int ringkb : {64, 128, 192}) {
        const int stage = seg * per;
        const int ring = ringkb * 1024 / stage;
        if (ring < 2 || stage > 64 * 1024 || ring * stage + 16 * ring + 64 > 227 * 1024) continue;
        const float us = timeit([&] { bulk_kernel<<<148, 288, ring * stage + 16 * ring + 64>>>(W, bytes, seg, ring, per, sink); });
        printf("{\"kind\": \"bulk\", \"seg\": %d, \"per_stage\": %d, \"ring\": %d, \"inflight_kb\": %d, \"us\": %.1f, \"GBps\": %.0f}\n",
               seg, per, ring, ring * stage / 1024, us, bytes / us / 1e3);
      }
  void* h = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &h, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)h;
  const int cols = 4096;
  const long long rows = bytes / (cols * 2);
  struct Box { int r, c; CUtensorMapSwizzle sw; };
  Box boxes[] = {{128, 64, CU_TENSOR_MAP_SWIZZLE_128B}, {64, 64, CU_TENSOR_MAP_SWIZZLE_128B}, {256, 64, CU_TENSOR_MAP_SWIZZLE_128B},
                 {16, 256, CU_TENSOR_MAP_SWIZZLE_NONE}, {32, 256, CU_TENSOR_MAP_SWIZZLE_NONE}, {64, 256, CU_TENSOR_MAP_SWIZZLE_NONE}};
  for (auto b : boxes) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)b.c, (cuuint32_t)b.r};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, b.sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", (int)r); continue; }
    const int stage = b.r * b.c * 2;
    for (int ringkb : {64, 128, 192}) {
      const int ring = ringkb * 1024 / stage;
      if (ring < 2) continue;
      const float us = timeit([&] { tmap_kernel<<<148, 288, ring * stage + 16 * ring + 64>>>(map, (int)rows, cols, b.r, b.c, ring, sink); });
      printf("{\"kind\": \"tmap\", \"box\": [%d, %d], \"ring\": %d, \"inflight_kb\": %d, \"us\": %.1f, \"GBps\": %.0f}\n", b.r,
             b.c, ring, ring * stage / 1024, us, bytes / us / 1e3);
    }
  }
  for (int blocks : {148 * 4, 148 * 8}) {
    const float us = timeit([&] { ldg_kernel<<<blocks, 256>>>((const uint4*)W, bytes / 16, sink); });
    printf("{\"kind\": \"ldg\", \"blocks\": %d, \"us\": %.1f, \"GBps\": %.0f}\n", blocks, us, bytes / us / 1e3);
  }
  const float us = timeit([&] { cudaMemcpyAsync(W + bytes / 2, W, bytes / 2, cudaMemcpyDeviceToDevice); });
  printf("{\"kind\": \"d2d_copy\", \"us\": %.1f, \"GBps_rw\": %.0f}\n", us, bytes / us / 1e3);
  return 0;
}
