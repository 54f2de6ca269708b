mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 300 python tools/profile_run.py --config mnist60k --iters 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r32_sym.csv timeout 600 python tools/profile_run.py --config mnist60k --iters 2 > /dev/null 2>&1
ls gpurun_out
