#!/bin/bash
# stage-1: max pass instantiations (registers), smem-staged next-batch walk, graph-replayed rounds
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_beam_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for gr in 1 0; do
      timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 --graph $gr >> gpurun_out/l_rounds.jsonl 2>> gpurun_out/l.err
    done
  done
done
timeout 600 python tools/draft_stage_probe.py > gpurun_out/l_draft_stage.json 2> gpurun_out/l_draft_stage.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 40 -o gpurun_out/l_tree_k8192 -f \
    python tools/tree_round_bench.py --V 32000 --K 8192 --B 1024 --builds 1 --graph 0 > gpurun_out/l_ncu_tree.log 2>&1
