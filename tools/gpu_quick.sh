#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_q.log 2>&1
timeout 600 python tools/gemm_bench.py --mode 0 --only 70b > gpurun_out/gb.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
