make -B > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sym or config2 or symmetric" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | tail -1; done
timeout 300 python tools/profile_run.py --config har200k --iters 10 2>&1 | tail -1
