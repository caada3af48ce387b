mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_gpu.py -x -q > gpurun_out/pytest_tp.log 2>&1
rm -f gpurun_out/gb_draft.txt
for M in 128 256; do for mode in 1 2; do for sched in 0 1 2 3; do
  echo "## M=$M mode=$mode sched=$sched" >> gpurun_out/gb_draft.txt
  timeout 300 python tools/gemm_bench.py --mode $mode --sched $sched --draft-m=$M --only 7b 2>&1 | grep 7b >> gpurun_out/gb_draft.txt
done; done; done
