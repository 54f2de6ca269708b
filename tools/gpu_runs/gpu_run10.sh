timeout 900 python tools/bench_configs.py --configs rings,har200k --iters 10 > gpurun_out/r10_cfg1.log 2>&1; cat gpurun_out/r10_cfg1.log | tail -3
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r10_cfg4.log 2>&1; tail -2 gpurun_out/r10_cfg4.log
timeout 300 python tools/profile_run.py --path mat --k 2 --iters 5 > gpurun_out/r10_k2.log 2>&1; tail -2 gpurun_out/r10_k2.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 100000 --iters 1 > gpurun_out/r10_splain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_stream" -c 1 -o gpurun_out/r10_sprof python tools/profile_run.py --path stream --config mnist1m --n 100000 --iters 1 > gpurun_out/r10_sncu.log 2>&1; tail -1 gpurun_out/r10_sncu.log
