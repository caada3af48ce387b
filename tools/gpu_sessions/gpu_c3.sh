#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_llama_gpu.py -q -x -p no:cacheprovider -k offload > gpurun_out/offload_test.log 2>&1
echo "rc=$?" >> gpurun_out/offload_test.log
timeout 1500 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1800 python bench.py --workload c3 --synthetic 4 --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_sharp20.json 2> gpurun_out/bench_c3_sharp20.err
