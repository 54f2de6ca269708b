mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream" 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 3 --path stream 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 3 --path stream --k 6 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config har200k --iters 3 --path stream 2>&1 | tail -1
timeout 300 python tools/profile_run.py --config har200k --iters 3 --path stream --k 10 2>&1 | tail -1
