#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp32_mode_gpu.py tests/test_named_configs_gpu.py -q -p no:cacheprovider -s --durations=10 > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
