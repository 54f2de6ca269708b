timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tiles" 2>&1 | tail -5 > gpurun_out/r6_tiles.log; cat gpurun_out/r6_tiles.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r6_pytest.log; cat gpurun_out/r6_pytest.log
timeout 300 python tools/bias_study.py > gpurun_out/r6_bias.log 2>&1; cat gpurun_out/r6_bias.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r6_bench.log 2>&1; tail -2 gpurun_out/r6_bench.log
