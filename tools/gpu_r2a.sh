#!/bin/bash
# round 2: new parity tests first (named configs, C2 replay, attention ws reuse), then the full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_named_configs_gpu.py tests/test_c2_replay_gpu.py -x -q -p no:cacheprovider -rA --durations=10 > gpurun_out/r2a_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_new.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r2a_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_all.log
