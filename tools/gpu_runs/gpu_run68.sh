timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric or mnist or config2 or rings" > gpurun_out/r68_pytest.log 2>&1; tail -2 gpurun_out/r68_pytest.log
for v in d1h1 d0h1 d0h0; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --iters 10 2>&1 | grep -E "a2 SpMM|J "
  timeout 300 ncu --kernel-name regex:spmm_sym --launch-skip 3 --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_elapsed.max \
    python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "duration|bytes|cycles"
done
