# round 2: every tensor-core kernel on the chained mainloop (chain.cuh: tc3 GEMM / self dots / full
# streaming, ssym): full GPU suite, smoke, bench, streaming speed
mkdir -p gpurun_out
make > gpurun_out/r2_07_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=8 --deselect tests/test_gpu_fullscale.py::test_full_size_objective_at_convergence > gpurun_out/r2_07_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r2_07_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k objective > gpurun_out/r2_07_jprec.log 2>&1; echo "jprec rc=$?"; grep -E "rel|passed|failed" gpurun_out/r2_07_jprec.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_07_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_07_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_07_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_07_bench.log | cut -c1-300
for v in "KKM_SSYM_BS=16" "KKM_SSYM_BS=16 KKM_CHAIN_KB=3"; do
  echo "== $v"; env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c150-330
done
timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream --symmetric off 2>&1 | tail -1 | cut -c150-330
