mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
timeout 600 python tools/gemm_probe.py > gpurun_out/probe2.txt 2>&1
for kpb in 1 2; do SX_GEMM_KPB=$kpb timeout 300 python tools/gemm_bench.py --mode 0 > gpurun_out/gb_auto_kpb$kpb.txt 2>&1; done
timeout 300 python tools/gemm_micro3.py > gpurun_out/micro3.txt 2>&1
