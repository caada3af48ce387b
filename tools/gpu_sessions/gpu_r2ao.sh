#!/bin/bash
# max pass with 256-thread CTAs (SX_TREE_MAX_PIPE=4) vs 128 (1): alternating, 3 reps
mkdir -p gpurun_out
for r in 1 2 3; do
  for p in 1 4; do
    for V in 32000 128256; do
      SX_TREE_MAX_PIPE=$p timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 | sed "s/^{/{\"pipe\": $p, /" >> gpurun_out/ao_rounds.jsonl 2>> gpurun_out/ao.err
    done
  done
done
SX_TREE_MAX_PIPE=4 timeout 600 python -m pytest tests/test_llama_gpu.py -x -q -p no:cacheprovider -k "large_tree or fused_round" > gpurun_out/ao_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ao_tests.log
