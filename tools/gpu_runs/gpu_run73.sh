make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore" > gpurun_out/r73_pytest.log 2>&1; tail -3 gpurun_out/r73_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 --kstore fp16 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 --kstore fp16x2 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config har200k --iters 10 --kstore fp16x2 2>&1 | tail -1
