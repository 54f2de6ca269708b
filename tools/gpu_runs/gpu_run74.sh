make > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none \
  -o gpurun_out/r74_spmm_tc python tools/profile_run.py --config mnist60k --iters 5 --kstore fp16 > gpurun_out/r74_ncu.log 2>&1; tail -1 gpurun_out/r74_ncu.log
