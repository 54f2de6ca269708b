make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore or symmetric or full_size" > gpurun_out/r81_pytest.log 2>&1; tail -2 gpurun_out/r81_pytest.log
for i in 1 2; do timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | grep "a2 SpMM"; done
timeout 300 python tools/profile_run.py --config har200k --iters 10 2>&1 | grep "a2 SpMM"
timeout 300 ncu --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "duration|bytes"
