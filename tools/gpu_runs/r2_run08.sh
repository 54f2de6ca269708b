# round 2: fixed-point scale for the f3 delta passes; Gaussian r^2 as (n_i - b) + (n_j - b); full suite
mkdir -p gpurun_out
make > gpurun_out/r2_08_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=5 --deselect tests/test_gpu_fullscale.py::test_full_size_objective_at_convergence > gpurun_out/r2_08_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2_08_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_08_pytest.log | head -20
timeout 900 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k objective > gpurun_out/r2_08_jprec.log 2>&1; echo "jprec rc=$?"; grep -E "rel|passed|failed" gpurun_out/r2_08_jprec.log
for v in "KKM_SSYM_BS=16" "KKM_SSYM_BS=8" "KKM_SSYM_BS=32"; do
  echo "== $v"; env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c150-330
done
echo "== 1M"; KKM_SSYM_BS=16 timeout 300 python tools/bench_configs.py --configs mnist1m --iters 2 2>&1 | tail -1 | cut -c150-330
