#!/bin/bash
# stage-1 update: sort-and-merge selection + lex merge (A/B with SX_TREE_MERGE=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_specinfer_gpu.py -x -q -p no:cacheprovider > gpurun_out/n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/n_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for m in 1 0; do
      SX_TREE_MERGE=$m timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 | sed "s/^{/{\"merge\": $m, /" >> gpurun_out/n_rounds.jsonl 2>> gpurun_out/n.err
    done
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 16 -o gpurun_out/n_tree_k8192 -f \
    python tools/tree_round_bench.py --V 32000 --K 8192 --B 1024 --builds 1 --graph 0 > gpurun_out/n_ncu_tree.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tree_ -c 12 -o gpurun_out/n_tree_k1024 -f \
    python tools/tree_round_bench.py --V 32000 --K 1024 --B 1024 --builds 1 --graph 0 > gpurun_out/n_ncu_tree1k.log 2>&1
