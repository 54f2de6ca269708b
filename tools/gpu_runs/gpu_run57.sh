make -B > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r57_pytest.log 2>&1; tail -2 gpurun_out/r57_pytest.log
timeout 900 python tools/j_precision.py --config har200k --iters 30 2>&1 | tail -1
timeout 900 python tools/j_precision.py --config mnist1m --n 200000 --iters 30 2>&1 | tail -1
