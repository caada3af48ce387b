#!/bin/bash
# GEMM split-tile plans as cooperative launches: GEMM / Llama tests, then the C2 step A/B-free check
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_llama_gpu.py tests/test_tp_gpu.py tests/test_named_configs_gpu.py -x -q -p no:cacheprovider > gpurun_out/aj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aj_tests.log
for r in 1 2 3; do
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --c3-steps 0 > gpurun_out/aj_bench_r$r.json 2> gpurun_out/aj_bench_r$r.err
done
