# round 2: a3 + a4 as one cooperative grid-wide launch (update_grid_kernel) on the 16-bit band paths;
# Dfull formed on demand. GPU suite, k = 10 / 32 timing, bench line
mkdir -p gpurun_out
make > gpurun_out/r2_27_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q --ignore=tests/test_multi_gpu.py > gpurun_out/r2_27_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_27_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_27_pytest.log | head
for kk in 10 32 10 32; do
  echo "== k=$kk"; timeout 600 python tools/bench_configs.py --configs mnist60k --k $kk --iters 100 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*\|"phases_ms_per_iter": {[^}]*}\|"final_J": [0-9.e+-]*' | tr '\n' ' '; echo
done
timeout 900 python bench.py --stream-iters 0 > gpurun_out/r2_27_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_27_bench.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:update_grid -c 3 python tools/profile_run.py --config mnist60k --iters 3 > gpurun_out/r2_27_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "duration" gpurun_out/r2_27_ncu.log
