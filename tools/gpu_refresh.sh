#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5-l3 > gpurun_out/bench_c5_l3.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload c4 > gpurun_out/bench_c4_1gpu.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --synthetic 4 > gpurun_out/bench_c2_sharp.json 2> gpurun_out/bench_sharp.err
