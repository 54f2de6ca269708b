cp gpurun_vars/libkkm_d0h1.so paper_2601_17136_b200/libkkm.so
timeout 600 ncu --set full --import-source on --kernel-name regex:spmm_sym --launch-skip 3 --launch-count 1 --clock-control none \
  -o gpurun_out/r67_sym_tail python tools/profile_run.py --config mnist60k --iters 5 > gpurun_out/r67_ncu.log 2>&1; tail -3 gpurun_out/r67_ncu.log
