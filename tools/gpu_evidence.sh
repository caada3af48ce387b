#!/bin/bash
# current-code evidence: GPU tests, C2 bench, launch list, ncu --set full per kernel family, C3, C5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_score|tree_row_stats|tree_update" -s 2 -c 6 -o gpurun_out/ncu_tree $B > gpurun_out/ncu_tree.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_attention" -s 200 -c 2 -o gpurun_out/ncu_attn $B > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"add_rmsnorm|rope_kv" -s 300 -c 4 -o gpurun_out/ncu_misc $B > gpurun_out/ncu_misc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kv_compact|verify_walk" -s 4 -c 4 -o gpurun_out/ncu_walk $B --synthetic 4 > gpurun_out/ncu_walk.log 2>&1
for s in 70b.qkv 70b.o 70b.gate_up_il 70b.down 7b.gate_up_il; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/ncu_gemm_$s python tools/gemm_one.py $s 0 >> gpurun_out/ncu_gemm.log 2>&1
done
timeout 1500 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c5-l3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
