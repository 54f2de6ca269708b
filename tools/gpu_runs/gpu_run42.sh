mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader
timeout 600 python tools/profile_run.py --config mnist1m --iters 2 --path stream 2>&1 | tail -1
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader
timeout 600 python tools/profile_run.py --config mnist1m --iters 2 --path stream --full-k 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 3 --path stream 2>&1 | tail -1
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 2>&1 | grep config | cut -c1-200
