make -B > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r49_pytest.log 2>&1; tail -2 gpurun_out/r49_pytest.log
timeout 900 python tools/bench_configs.py --configs rings,mnist60k --iters 30 2>&1 | grep config | cut -c1-330
