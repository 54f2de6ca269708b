set -x
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -k "tiles and bf16x3" 2>&1 | tail -30 > gpurun_out/r2_tiles.log; cat gpurun_out/r2_tiles.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2_pytest.log; cat gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -3 gpurun_out/r2_smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench.log 2>&1; tail -3 gpurun_out/r2_bench.log
