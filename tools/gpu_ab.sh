#!/bin/bash
mkdir -p gpurun_out
for w in "" "--synthetic 4"; do
  for a in mma auto mma auto; do
    echo "== $w --attn $a" >> gpurun_out/ab.log
    timeout 600 python bench.py $w --attn $a --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/ab.log
  done
done
