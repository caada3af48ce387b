#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
SX_GEMM_PDL=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_nopdl.json 2> gpurun_out/bench_c2_nopdl.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_b.json 2> gpurun_out/bench_c2_b.err
