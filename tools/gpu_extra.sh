#!/bin/bash
# extra configurations: C4 shape on one GPU (K=4096), C3 and C2 with the synthetic shared bias (sharp variant)
mkdir -p gpurun_out
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_1gpu.json 2> gpurun_out/bench_c4_1gpu.err
timeout 900 python bench.py --synthetic 4 --no-cpu-baseline > gpurun_out/bench_c2_sharp.json 2> gpurun_out/bench_c2_sharp.err
timeout 1500 python bench.py --workload c3 --synthetic 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_sharp.json 2> gpurun_out/bench_c3_sharp.err
