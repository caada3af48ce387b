// Thin-batch (M <= kGemvMaxTokens) projection path of sx_gemm_bf16 / sx_gemm_qkv_rope (gemv.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sx {

constexpr int kGemvMaxTokens = 4;

struct GemvArgs {
  const __nv_bfloat16* W;
  const __nv_bfloat16* X;
  void* out;
  long long ldo;
  int M, Nf, K, epi;
  const int* rope_pos;
  const int* rope_slot;
  int rope_pos_base, rope_slot_base, rope_H, rope_KVH;
  const float* rope_cos;
  const float* rope_sin;
  __nv_bfloat16* rope_q;
  __nv_bfloat16* rope_kc;
  __nv_bfloat16* rope_vc;
  long long rope_slots;
};

bool gemv_applies(int M, int epi, int dual);
int launch_gemv(const GemvArgs& g, cudaStream_t stream);

}  // namespace sx
