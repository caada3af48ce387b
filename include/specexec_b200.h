/*
 * specexec_b200.h -- C ABI of the B200-native SpecExec hot path.
 *
 * The reference (`speckit`, pure Python + numpy) has no native boundary: its
 * hot path is the Python call chain
 *   generate_specexec  pkg/src/speckit/engine.py:92-131
 *     precompute       pkg/src/speckit/engine.py:73-89
 *       build_sssp     pkg/src/speckit/tree.py:240-327
 *       LanguageModel.next_distributions  pkg/src/speckit/models.py:47-52
 *     apply_warp/sample pkg/src/speckit/sampling.py:66-113
 * The entry points below are what a ctypes binding of that chain calls (see
 * INTEGRATION.md). Each one names the reference interface whose semantics it
 * implements.
 *
 * Conventions
 *  - Device buffers are allocated by the caller (PyTorch) and passed as raw
 *    pointers plus explicit sizes; kernels never allocate or free.
 *  - Every call is asynchronous on the given stream (cudaStream_t; NULL = the
 *    legacy default stream) unless documented otherwise.
 *  - Return: 0 ok; < 0 argument error (the Python layer raises ValueError);
 *    > 0 a cudaError_t (RuntimeError). sx_last_error() returns a thread-local
 *    message for the last failure on the calling thread.
 *  - No global mutable state besides the thread-local error string and an
 *    internal cache of TMA descriptors (mutex-protected).
 */
#ifndef SPECEXEC_B200_H_
#define SPECEXEC_B200_H_

#include <stdint.h>
#include <cuda_runtime.h>

#if defined(__GNUC__)
#define SX_API __attribute__((visibility("default")))
#else
#define SX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- misc */
SX_API int sx_abi_version(void);
SX_API const char* sx_last_error(void);

/* ----------------------------------------------- KG: dense projections
 * Y[t, f] (op)= sum_k X[t, k] * W[f, k]; bf16 in, fp32 accumulate on tcgen05.
 * Replaces the dense part of LanguageModel.next_distributions
 * (pkg/src/speckit/models.py:47-52) for Llama-shaped models.
 *   W   [N, K] bf16 row-major (nn.Linear weight layout)
 *   W2  optional second weight [N, K] (SwiGLU up-projection) or NULL
 *   X   [M, K] bf16 row-major, contiguous
 *   out [M, ldo] bf16 or fp32 depending on the epilogue
 *   ws  fp32 split-K workspace (sx_gemm_plan reports the size), may be NULL
 *       when no split is needed. splits_req <= 0 picks automatically.
 */
enum {
  SX_EPI_BF16 = 0,        /* out bf16  = acc                       */
  SX_EPI_F32 = 1,         /* out fp32  = acc                       */
  SX_EPI_ADD_F32 = 2,     /* out fp32 += acc (residual stream)     */
  SX_EPI_SWIGLU_BF16 = 3  /* out bf16  = silu(acc(W)) * acc(W2)    */
};
SX_API int sx_gemm_plan(int M, int N, int K, int dual, int splits_req, int* bn_out, int* splits_out,
                 long long* ws_floats_out);
SX_API int sx_gemm_bf16(const void* W, const void* W2, const void* X, void* out, float* ws, long long ws_floats,
                 int M, int N, int K, long long ldo, int epi, int splits_req, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECEXEC_B200_H_ */
