#!/bin/bash
# GEMM programmatic dependent launch A/B in the full C2 step (alternating, two runs each; no C3 / CPU legs)
mkdir -p gpurun_out
for r in 1 2 3 4 5 6; do
  for p in 0 1; do
    SX_GEMM_PDL=$p timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/ae_pdl${p}_r$r.json 2> gpurun_out/ae_pdl${p}_r$r.err
  done
done
