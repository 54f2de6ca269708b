# re-entry validation on a fresh box: GPU tests, smoke, the default bench line, the reference arm,
# and the launch list of the bench (ncu, after the plain run exited 0)
mkdir -p gpurun_out
make > gpurun_out/r106_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r106_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r106_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r106_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r106_smoke.log
timeout 600 python bench.py > gpurun_out/r106_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r106_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r106_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r106_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r106_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r106_ncu.log 2>&1; echo "ncu rc=$?"
