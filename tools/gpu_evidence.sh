#!/bin/bash
# ncu evidence for each kernel family + C3 offload + acceptance sweep (one GPU).
mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_score|tree_row_stats|tree_update" -s 3 -c 3 -o gpurun_out/ncu_tree $B > gpurun_out/ncu_tree.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attention -s 300 -c 2 -o gpurun_out/ncu_attn $B > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kv_compact|verify_walk|add_rmsnorm" -s 10 -c 4 -o gpurun_out/ncu_misc $B > gpurun_out/ncu_misc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/ncu_gemm_qkv python tools/gemm_one.py 70b.qkv 0 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/ncu_gemm_gateup python tools/gemm_one.py 70b.gate_up 0 >> gpurun_out/ncu_gemm.log 2>&1
timeout 900 python tools/acceptance_sweep.py --draft llama2-7b --target llama2-70b --budgets 64,256,1024,2048 --seeds 1 --tokens 32 --synthetic 4 --out gpurun_out/acceptance_c2.jsonl > gpurun_out/acceptance_c2.log 2>&1
timeout 1200 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
