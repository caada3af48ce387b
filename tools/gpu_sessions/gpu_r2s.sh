#!/bin/bash
# stage-1 max pass: TMA ring with >= 4 units per CTA vs register double buffer
mkdir -p gpurun_out
SX_TREE_MAX_PIPE=3 timeout 900 python -m pytest tests/tess_tree_gpu.py tests/tess_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s_tests.log
for V in 32000 128256; do
  for K in 1024 8192; do
    for p in 1 3; do
      SX_TREE_MAX_PIPE=$p timeout 300 python tools/tree_round_bench.py --V $V --K $K --B 1024 | sed "s/^{/{\"pipe\": $p, /" >> gpurun_out/s_rounds.jsonl 2>> gpurun_out/s.err
    done
  done
done
SX_TREE_MAX_PIPE=3 timeout 600 ncu --set full --clock-control none -k regex:tree_rows_max -c 4 -o gpurun_out/s_max -f \
    python tools/tree_round_bench.py --V 32000 --K 8192 --B 1024 --builds 1 --graph 0 > gpurun_out/s_ncu.log 2>&1
