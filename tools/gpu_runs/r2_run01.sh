# round 2: quick fixes (per-device smem opt-in, finalize for large k, opt-in peer exchange without
# trap) + the full-scale oracle parity tests; GPU suite, smoke, bench
mkdir -p gpurun_out
make > gpurun_out/r2_01_make.log 2>&1 || { echo make failed; tail gpurun_out/r2_01_make.log; exit 1; }
nproc
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2_01_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2_01_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_01_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_01_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_01_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_01_bench.log | cut -c1-600
