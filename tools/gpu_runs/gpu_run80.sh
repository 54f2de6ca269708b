for v in p0 p1 p3 p0 p1 p3; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | grep "a2 SpMM"
done
cp gpurun_vars/libkkm_p1.so paper_2601_17136_b200/libkkm.so
timeout 300 ncu --kernel-name regex:spmm_tc --launch-skip 3 --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "duration|bytes"
