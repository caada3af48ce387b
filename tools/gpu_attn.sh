#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "test rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/attn_probe.py > gpurun_out/attn_probe.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --synthetic 4 > gpurun_out/bench_c2_sharp.json 2> gpurun_out/bench_c2_sharp.err
