#!/bin/bash
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -x -q -p no:cacheprovider > gpurun_out/attn_test.log 2>&1
echo "test rc=$?" >> gpurun_out/attn_test.log
timeout 300 python tools/attn_probe.py > gpurun_out/attn_probe.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attention -c 2 -o gpurun_out/ncu_attn_tc_final python tools/attn_one.py 64 8 1025 130 2 2 > gpurun_out/ncu_attn_tc_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launch_bench.log 2>&1
