#!/bin/bash
# stage-1: fused exact pass (sum + score in one persistent grid with per-row readiness flags) A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfer_gpu.py tests/test_llama_gpu.py tests/test_c2_replay_gpu.py -x -q -p no:cacheprovider > gpurun_out/v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for f in 1 0; do
      SX_TREE_FUSED_EXACT=$f timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 | sed "s/^{/{\"fused_exact\": $f, /" >> gpurun_out/v_rounds.jsonl 2>> gpurun_out/v.err
    done
  done
done
timeout 600 ncu --set full --clock-control none -k regex:tree_ -c 12 -o gpurun_out/v_tree_k1024 -f \
    python tools/tree_round_bench.py --V 32000 --K 1024 --B 1024 --builds 1 --graph 0 > gpurun_out/v_ncu_tree1k.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tree_ -c 12 -o gpurun_out/v_tree_v128k -f \
    python tools/tree_round_bench.py --V 128256 --K 1024 --B 1024 --builds 1 --graph 0 > gpurun_out/v_ncu_tree128k.log 2>&1
