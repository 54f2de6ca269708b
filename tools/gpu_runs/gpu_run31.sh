mkdir -p gpurun_out
make -B > gpurun_out/r31_build.log 2>&1 || { tail -20 gpurun_out/r31_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r31_pytest.log 2>&1; tail -3 gpurun_out/r31_pytest.log
for a in "" "--full-k"; do timeout 300 python tools/profile_run.py --config mnist60k --iters 10 $a 2>&1 | tail -3; done
timeout 300 python tools/profile_run.py --config har200k --iters 5 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r31_bench.log 2>&1; tail -1 gpurun_out/r31_bench.log | cut -c1-400
