#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention -s 2 -c 1 -o gpurun_out/an_attn_draft -f python tools/attn_one.py 32 32 1023 160 2 0 > gpurun_out/an.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention -s 2 -c 1 -o gpurun_out/an_attn_c2 -f python tools/attn_one.py 64 8 1025 130 2 0 >> gpurun_out/an.log 2>&1
