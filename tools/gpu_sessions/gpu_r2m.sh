#!/bin/bash
# round-2 evidence at HEAD: driver sequence (tests, smoke, both bench arms), launch list of the C2 step,
# ncu --set full of the 70B target-pass GEMM shapes (roofline.traffic), the stage-1 kernels and the one-token GEMV
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/m_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/m_smoke.log
timeout 1200 python bench.py --impl reference > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/m_bench_ncu.log 2>&1
for s in 70b.qkv 70b.o 70b.gate_up_il 70b.down 7b.gate_up_il; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/m_ncu_gemm_$s python tools/gemm_one.py $s 0 >> gpurun_out/m_ncu_gemm.log 2>&1
done
timeout 600 python tools/profile_step.py --json gpurun_out/m_profile_step.json > gpurun_out/m_profile_step.txt 2>&1
