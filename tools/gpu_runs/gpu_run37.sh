mkdir -p gpurun_out
make -B > gpurun_out/r37_build.log 2>&1 || { tail -20 gpurun_out/r37_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r37_pytest.log 2>&1; tail -3 gpurun_out/r37_pytest.log
for a in "" "--full-k"; do timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 3 --path stream $a 2>&1 | tail -1; done
for a in "" "--full-k"; do timeout 300 python tools/profile_run.py --config har200k --iters 3 --path stream $a 2>&1 | tail -1; done
timeout 600 python tools/profile_run.py --config mnist1m --iters 2 --path stream 2>&1 | tail -1
