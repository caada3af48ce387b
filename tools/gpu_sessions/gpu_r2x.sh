#!/bin/bash
# deep-tree parity test + ncu of the tree attention on the C2 target-pass and draft shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tree_gpu.py -x -q -p no:cacheprovider -k "deep or sssp or uniform" > gpurun_out/x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/x_tests.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention -s 2 -c 1 -o gpurun_out/x_attn_c2 -f python tools/attn_one.py 64 8 1025 130 2 0 > gpurun_out/x_attn.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention -s 2 -c 1 -o gpurun_out/x_attn_draft -f python tools/attn_one.py 32 32 1024 160 3 0 >> gpurun_out/x_attn.log 2>&1
timeout 300 python tools/attn_one.py 64 8 1025 130 2 0 >> gpurun_out/x_attn.log 2>&1
timeout 300 python tools/attn_one.py 32 32 1024 160 3 0 >> gpurun_out/x_attn.log 2>&1
