# finalize: the last five levels of the fixed block tree as warp shuffles (same pairs, same bits):
# GPU tests, the bench line (final J must be bitwise the earlier 69087744.09652902), launch list
mkdir -p gpurun_out
make > /dev/null 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r111_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r111_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r111_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r111_smoke.log
timeout 600 python bench.py > gpurun_out/r111_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r111_bench.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['phases_ms_per_step'],d['clocks'],d['final_J'],d['roofline']['frac'])"
