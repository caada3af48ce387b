#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5-l3 > gpurun_out/bench_c5_l3.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload c4 > gpurun_out/bench_c4_1gpu.json 2> gpurun_out/bench_c4.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention_tc -c 1 -o gpurun_out/ncu_attn_split python tools/attn_one.py 64 8 1 2000 0 0 > gpurun_out/ncu_attn_split.log 2>&1
