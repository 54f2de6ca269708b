make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore or symmetric or sym or full_size" > gpurun_out/r87_pytest.log 2>&1; tail -1 gpurun_out/r87_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "a1 GEMM|a2 SpMM"
timeout 300 python tools/profile_run.py --config mnist60k --iters 5 --kstore fp32 2>&1 | grep -E "a1 GEMM"
timeout 300 python tools/profile_run.py --config har200k --iters 3 2>&1 | grep -E "a1 GEMM|a2 SpMM"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/run_multi.py > gpurun_out/r87_multi2.log 2>&1; grep -E "MULTI" gpurun_out/r87_multi2.log
