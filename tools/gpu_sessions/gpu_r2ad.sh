#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_stage1_variants_gpu.py -x -q -p no:cacheprovider > gpurun_out/ad_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ad_tests.log
