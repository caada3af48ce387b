#!/bin/bash
# in-loop A/B: CTA-pair tiles wherever legal (SX_GEMM_PAIR_MODE=2) vs the planner's auto choice
mkdir -p gpurun_out
for r in 4 5 6 7; do
  for m in 0 2; do
    SX_GEMM_PAIR_MODE=$m timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/ar_pm${m}_r$r.json 2> gpurun_out/ar_pm${m}_r$r.err
  done
done
