# ncu --set full of the a3 (finalize, int64 S in, last block finishes c and J) and a4 (assign) kernels, config 2
mkdir -p gpurun_out
make > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --kernel-name regex:"finalize|assign_kernel" --launch-skip 6 --launch-count 2 --clock-control none \
  -o gpurun_out/r107_a3a4 python tools/profile_run.py --config mnist60k --iters 6 > gpurun_out/r107_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r107_ncu.log
