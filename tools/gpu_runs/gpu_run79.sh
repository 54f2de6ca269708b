make > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none \
  -o gpurun_out/r79_spmm_tc_x2 python tools/profile_run.py --config mnist60k --iters 5 > gpurun_out/r79_ncu.log 2>&1; tail -1 gpurun_out/r79_ncu.log
