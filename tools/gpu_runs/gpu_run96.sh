make > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --kernel-name regex:"finalize|assign_kernel" --launch-skip 6 --launch-count 2 --clock-control none \
  -o gpurun_out/r96_a3a4 python tools/profile_run.py --config mnist60k --iters 6 > gpurun_out/r96_ncu.log 2>&1; tail -1 gpurun_out/r96_ncu.log
