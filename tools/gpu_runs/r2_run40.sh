# round 2: band GEMM epilogue with direct 16-byte stores of the fp16 planes (no TMA staging chain);
# parity (16-bit band tests), config-2 GEMM time (bench_configs a1_roofline) x3, ncu of the GEMM
mkdir -p gpurun_out
make > gpurun_out/r2_40_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py tests/test_gpu_fullscale.py -m gpu -x -q -k "kx2 or kstore or fp16 or config3 or objective" > gpurun_out/r2_40_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_40_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_40_pytest.log | head
for r in 1 2 3; do
  timeout 600 python tools/bench_configs.py --configs mnist60k --iters 20 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*\|"init_s": [0-9.]*\|"a1_roofline": {[^}]*}\|"final_J": [0-9.e+-]*' | tr '\n' ' '; echo
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc3_gemm -c 1 python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r2_40_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "duration|dram|tensor|per_second" gpurun_out/r2_40_ncu.log
