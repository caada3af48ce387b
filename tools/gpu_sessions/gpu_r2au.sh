#!/bin/bash
# run-to-run spread of the C2 step at HEAD (10 back-to-back runs of the timed loop)
mkdir -p gpurun_out
for r in $(seq 1 10); do
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/au_r$r.json 2>/dev/null
done
