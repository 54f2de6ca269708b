mkdir -p gpurun_out
make -B > gpurun_out/r47_build.log 2>&1 || { tail -20 gpurun_out/r47_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kpp.py -x -q > gpurun_out/r47_pytest.log 2>&1; tail -25 gpurun_out/r47_pytest.log
