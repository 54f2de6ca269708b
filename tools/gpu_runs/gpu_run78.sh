make > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r78_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r78_ncu_bench.log 2>&1; tail -1 gpurun_out/r78_ncu_bench.log | cut -c1-100
python tools/ncu_summary.py --launches gpurun_out/r78_launches.csv | head -16
timeout 600 ncu --set full --import-source on --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none \
  -o gpurun_out/r78_spmm_tc_x2 python tools/profile_run.py --config mnist60k --iters 5 > gpurun_out/r78_ncu.log 2>&1; tail -1 gpurun_out/r78_ncu.log
