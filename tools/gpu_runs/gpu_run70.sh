make > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_kstore.py -x -q > gpurun_out/r70_pytest.log 2>&1; tail -30 gpurun_out/r70_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 --kstore fp16 2>&1 | tail -3
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | tail -1
