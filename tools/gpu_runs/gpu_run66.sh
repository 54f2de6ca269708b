# variants of the fused column-sum spmm_sym (discard x L2 hints): a2 time and DRAM bytes
for v in d1h1 d0h1 d0h0 d1h0; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --iters 10 2>&1 | grep "a2 SpMM"
  timeout 300 ncu --kernel-name regex:spmm_sym --launch-skip 3 --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    python tools/profile_run.py --config mnist60k --iters 5 2>&1 | grep -E "duration|bytes"
done
