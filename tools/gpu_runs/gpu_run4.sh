timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/r4_pytest.log; cat gpurun_out/r4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4_smoke.log 2>&1; tail -3 gpurun_out/r4_smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r4_bench.log 2>&1; tail -3 gpurun_out/r4_bench.log
