#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_llama_gpu.py -x -q -p no:cacheprovider -k "large_tree" > gpurun_out/ak_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ak_tests.log
