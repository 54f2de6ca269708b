make -B > /dev/null 2>&1 || exit 1
timeout 300 python tools/profile_run.py --config mnist60k --iters 12 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed.sum --clock-control none -k regex:spmm_sym --csv --log-file gpurun_out/r53_sym.csv python tools/profile_run.py --config mnist60k --iters 12 > /dev/null 2>&1; echo "exit $?"
