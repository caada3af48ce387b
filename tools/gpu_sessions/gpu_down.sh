#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/gemm_plan_sweep.py --set c2 --only 70b.down --fine --out gpurun_out/plan_fine_down.jsonl > gpurun_out/plan_fine_down.txt 2>&1
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-sequential 2>/dev/null | tail -1 > gpurun_out/bench_down_$i.json
done
