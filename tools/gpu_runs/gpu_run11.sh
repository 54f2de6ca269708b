timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "tiles and fp16x3 and mnist" 2>&1 | tail -3 > gpurun_out/r11_tiles.log; cat gpurun_out/r11_tiles.log
if grep -q passed gpurun_out/r11_tiles.log; then
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r11_pytest.log; cat gpurun_out/r11_pytest.log
timeout 300 python tools/profile_run.py --path mat --iters 3 > gpurun_out/r11_mat.log 2>&1; tail -2 gpurun_out/r11_mat.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 3 > gpurun_out/r11_stream.log 2>&1; tail -1 gpurun_out/r11_stream.log
timeout 300 python tools/bias_study.py > gpurun_out/r11_bias.log 2>&1; grep fp16 gpurun_out/r11_bias.log
fi
