#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python bench.py --workload c3 --synthetic 4 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_sharp20.json 2> gpurun_out/bench_c3_sharp20.err
timeout 1200 python bench.py --synthetic 4 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_sharp20.json 2> gpurun_out/bench_c2_sharp20.err
