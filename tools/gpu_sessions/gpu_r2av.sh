#!/bin/bash
# flakiness check: the GPU suite twice more at HEAD
mkdir -p gpurun_out
for r in 1 2; do
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/av_tests_r$r.log 2>&1; echo "rc=$?" >> gpurun_out/av_tests_r$r.log
done
