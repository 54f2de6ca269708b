timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r8_pytest.log; cat gpurun_out/r8_pytest.log
timeout 300 python tools/bias_study.py > gpurun_out/r8_bias.log 2>&1; grep fp16 gpurun_out/r8_bias.log
timeout 300 python tools/profile_run.py --path mat > gpurun_out/r8_mat.log 2>&1; tail -1 gpurun_out/r8_mat.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 3 > gpurun_out/r8_stream.log 2>&1; tail -2 gpurun_out/r8_stream.log
