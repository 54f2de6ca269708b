mkdir -p gpurun_out
make -B > gpurun_out/r44_build.log 2>&1 || { tail -20 gpurun_out/r44_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "incremental" > gpurun_out/r44_pytest.log 2>&1; tail -15 gpurun_out/r44_pytest.log
timeout 600 python tools/inc_bench.py --config mnist60k 2>&1 | tail -1 | cut -c1-900
timeout 600 python tools/inc_bench.py --config mnist60k --n 200000 --iters 30 --path stream 2>&1 | tail -1 | cut -c1-900
