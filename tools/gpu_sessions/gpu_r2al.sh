#!/bin/bash
# KV1 argmax keys for the TP target at t=0: TP tests (thread ranks, 2 processes), walk tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tp_gpu.py tests/test_tp_procs_gpu.py tests/test_tree_gpu.py tests/test_plugin_boundary_gpu.py -x -q -p no:cacheprovider > gpurun_out/al_tests.log 2>&1; echo "rc=$?" >> gpurun_out/al_tests.log
