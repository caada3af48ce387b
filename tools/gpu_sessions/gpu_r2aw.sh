#!/bin/bash
# root-round lex ranks by token bitmap: tree / replay / variant tests, then per-round timing (root rounds)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfer_gpu.py tests/test_stage1_variants_gpu.py tests/test_plugin_boundary_gpu.py -x -q -p no:cacheprovider > gpurun_out/aw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aw_tests.log
timeout 900 python -m pytest tests/test_llama_gpu.py -x -q -p no:cacheprovider -k "large_tree or fused_round or replay" >> gpurun_out/aw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aw_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 >> gpurun_out/aw_rounds.jsonl 2>> gpurun_out/aw.err
  done
done
