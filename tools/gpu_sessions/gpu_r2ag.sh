#!/bin/bash
# in-loop (power-capped) A/B of GEMM planner knobs on the C2 step, alternating with the default
mkdir -p gpurun_out
run() { timeout 600 env $1 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/ag_$2_r$3.json 2> gpurun_out/ag_$2_r$3.err; }
for r in 1 2 3; do
  run "X=0" base $r
  run "SX_GEMM_STAGES=6" st6 $r
  run "SX_GEMM_STAGES=12" st12 $r
  run "SX_GEMM_KPB=1" kpb1 $r
  run "SX_ATTN_ANC_CUDA=0" anc0 $r
done
