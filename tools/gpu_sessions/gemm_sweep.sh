#!/bin/bash
# tile / pipeline sweep of the 70B target-pass projections (tools/gemm_bench.py per setting)
for mode in 1 0; do
for cap in 128 192 256; do
for st in 4 8; do
  echo "== mode=$mode bn_cap=$cap stages=$st"
  SX_GEMM_BN_CAP=$cap SX_GEMM_STAGES=$st python tools/gemm_bench.py --mode $mode 2>&1 | grep 70b
done; done; done
