#!/bin/bash
# draft-shape attention A/B (MHA, A = 2 / 3 / 17) + GQA guard
mkdir -p gpurun_out
for f in 1 0; do
  for c in "32 32 1023 160 2" "32 32 1023 160 3" "32 32 1024 160 17" "64 8 1025 130 17" "64 8 1025 130 2"; do
    echo "anc_cuda=$f $c $(SX_ATTN_ANC_CUDA=$f timeout 120 python tools/attn_one.py $c 0 2>&1 | tail -1)" >> gpurun_out/ab_attn.txt
  done
done
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
