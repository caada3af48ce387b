#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_offload_gpu.py tests/test_plugin_boundary_gpu.py tests/test_fp32_mode_gpu.py -q -p no:cacheprovider -s --durations=10 > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_b200.json 2> gpurun_out/r2d_b200.err
