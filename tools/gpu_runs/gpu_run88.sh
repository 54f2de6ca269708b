make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore or symmetric" > gpurun_out/r88_pytest.log 2>&1; tail -1 gpurun_out/r88_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 10 2>&1 | grep -E "a1 GEMM|a2 SpMM"
timeout 300 python tools/profile_run.py --config har200k --iters 5 2>&1 | grep -E "a1 GEMM|a2 SpMM"
