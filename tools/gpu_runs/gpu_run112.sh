# fused_update (single-CTA a3 + a4, config 1): the same shuffle tail of the fixed tree; GPU tests and config 1
mkdir -p gpurun_out
make > /dev/null 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r112_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r112_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r112_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r112_smoke.log
timeout 600 python tools/bench_configs.py --configs rings > gpurun_out/r112_cfg1.log 2>&1; echo "cfg1 rc=$?"; tail -2 gpurun_out/r112_cfg1.log | cut -c1-300
