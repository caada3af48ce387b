#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/ac_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ac_tests.log
