mkdir -p gpurun_out
make -B > gpurun_out/r34_build.log 2>&1 || { tail -20 gpurun_out/r34_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r34_pytest.log 2>&1; tail -2 gpurun_out/r34_pytest.log
for a in "" "--full-k"; do timeout 300 python tools/profile_run.py --config mnist60k --iters 10 $a 2>&1 | tail -2; done
timeout 300 python tools/profile_run.py --config har200k --iters 5 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r34_sym.csv timeout 600 python tools/profile_run.py --config mnist60k --iters 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmm_sym -c 1 -o gpurun_out/r34_spmm_sym timeout 600 python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r34_ncu.log 2>&1; tail -2 gpurun_out/r34_ncu.log
