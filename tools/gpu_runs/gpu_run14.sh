timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "rings and stream" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r14_pytest.log; cat gpurun_out/r14_pytest.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 2 > gpurun_out/r14_stream.log 2>&1; tail -1 gpurun_out/r14_stream.log
timeout 300 python tools/profile_run.py --path stream --config har200k --n 200000 --iters 2 > gpurun_out/r14_streamh.log 2>&1; tail -1 gpurun_out/r14_streamh.log
timeout 300 python tools/profile_run.py --path mat --iters 5 > gpurun_out/r14_mat.log 2>&1; tail -2 gpurun_out/r14_mat.log
timeout 300 python tools/profile_run.py --path mat --iters 5 --k 2 > gpurun_out/r14_mat2.log 2>&1; tail -1 gpurun_out/r14_mat2.log
timeout 300 python tools/profile_run.py --path mat --config har200k --n 100000 --iters 5 > gpurun_out/r14_har.log 2>&1; tail -1 gpurun_out/r14_har.log
