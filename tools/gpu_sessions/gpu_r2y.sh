#!/bin/bash
# one-token rounds: GEMV ring depth 3 (two CTAs / SM) vs 4
mkdir -p gpurun_out
for s in 4 3; do
  SX_GEMV_STAGES=$s timeout 300 python tools/draft_probe.py --rows 1 > gpurun_out/y_probe7b_s$s.txt 2>&1
  SX_GEMV_STAGES=$s timeout 600 python tools/draft_probe.py --model llama2-70b --rows 1 > gpurun_out/y_probe70b_s$s.txt 2>&1
done
