#!/bin/bash
# offloaded target: accepted tokens and tokens/s vs budget (the pass cost is budget-independent until compute-bound)
mkdir -p gpurun_out
rm -f gpurun_out/c3_budget.jsonl
for K in 512 2048 8192; do
  timeout 1500 python bench.py --workload c3 --synthetic 4 --budget $K --steps 10 --no-cpu-baseline --no-e2e $( [ $K != 512 ] && echo --no-sequential ) 2>/dev/null | tail -1 >> gpurun_out/c3_budget.jsonl
done
