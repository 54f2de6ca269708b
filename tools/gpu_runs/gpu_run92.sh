make > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r92_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r92_ncu_bench.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/r92_launches.csv | head -12
timeout 600 ncu --set full --import-source on --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none \
  -o gpurun_out/r92_spmm_tc python tools/profile_run.py --config mnist60k --iters 5 > gpurun_out/r92_ncu.log 2>&1; tail -1 gpurun_out/r92_ncu.log
timeout 600 ncu --set full --kernel-name regex:tc2_gemm --launch-count 1 --clock-control none \
  -o gpurun_out/r92_gemm python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r92_ncu_gemm.log 2>&1; tail -1 gpurun_out/r92_ncu_gemm.log
