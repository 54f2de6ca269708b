timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "rings and stream" 2>&1 | tail -3 > gpurun_out/r12_t.log; cat gpurun_out/r12_t.log
if grep -q passed gpurun_out/r12_t.log; then
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r12_pytest.log; cat gpurun_out/r12_pytest.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 3 > gpurun_out/r12_stream.log 2>&1; tail -1 gpurun_out/r12_stream.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 100000 --iters 1 > gpurun_out/r12_splain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc2_" -c 1 -o gpurun_out/r12_sprof python tools/profile_run.py --path stream --config mnist1m --n 100000 --iters 1 > gpurun_out/r12_sncu.log 2>&1; tail -1 gpurun_out/r12_sncu.log
fi
