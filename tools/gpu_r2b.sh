#!/bin/bash
# round 2: named-config parity (bf16-policy oracle), plugin boundary, then both bench arms
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_named_configs_gpu.py tests/test_plugin_boundary_gpu.py -q -p no:cacheprovider -s --durations=10 > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
timeout 900 python bench.py --steps 6 --warmup 3 > gpurun_out/r2b_b200.json 2> gpurun_out/r2b_b200.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
