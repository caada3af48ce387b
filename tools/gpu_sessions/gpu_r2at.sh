#!/bin/bash
# in-loop A/B under the power cap: attention kernel choice and token-tile cap
mkdir -p gpurun_out
B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0"
for r in 1 2 3 4; do
  timeout 600 $B > gpurun_out/at_base_r$r.json 2>/dev/null
  timeout 600 $B --attn mma > gpurun_out/at_mma_r$r.json 2>/dev/null
  SX_GEMM_BN_CAP=192 timeout 600 $B > gpurun_out/at_bn192_r$r.json 2>/dev/null
done
