#!/bin/bash
mkdir -p gpurun_out
for b in 128 512 1024; do
  timeout 600 python bench.py --batch $b --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_b$b.json 2> gpurun_out/bench_b$b.err
done
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1200 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python tools/gemm_plan_sweep.py --set c2 --out gpurun_out/plan_sweep_c2.jsonl > gpurun_out/plan_sweep_c2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
