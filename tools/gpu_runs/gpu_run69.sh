timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric or mnist or config2 or rings" > gpurun_out/r69_pytest.log 2>&1; tail -1 gpurun_out/r69_pytest.log
for v in old h0 h1 old h0 h1; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | grep -E "a2 SpMM|phases" | cut -c1-60,180-400
done
for v in old h1; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  timeout 300 ncu --kernel-name regex:spmm_sym --launch-skip 3 --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_elapsed.max \
    python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "duration|bytes|cycles"
done
