#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_procs_gpu.py tests/test_abi.py -x -q -p no:cacheprovider > gpurun_out/am_tests.log 2>&1; echo "rc=$?" >> gpurun_out/am_tests.log
