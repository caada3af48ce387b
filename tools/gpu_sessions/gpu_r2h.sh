#!/bin/bash
# HEAD re-validation after the container restore: all GPU tests, smoke, stage-1 rounds + ncu (V=32000/128256),
# draft probe + gemv ncu, the C2 bench and the tree/GEMM launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
for V in 32000 128256; do
  timeout 300 python tools/tree_round_bench.py --V $V --K 1024 --B 1024 >> gpurun_out/h_rounds.jsonl 2>> gpurun_out/h.err
  timeout 300 python tools/tree_round_bench.py --V $V --K 8192 --B 1024 >> gpurun_out/h_rounds.jsonl 2>> gpurun_out/h.err
done
timeout 600 python tools/draft_probe.py --rows 1,1024 > gpurun_out/h_draft_probe.txt 2>&1
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
for V in 32000 128256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 12 -o gpurun_out/h_tree_v$V -f \
    python tools/tree_round_bench.py --V $V --K 1024 --B 1024 --builds 1 > gpurun_out/h_ncu_tree_v$V.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -c 6 -o gpurun_out/h_gemv -f \
  python tools/draft_probe.py --rows 1 --iters 1 --ctx 100 > gpurun_out/h_ncu_gemv.log 2>&1
