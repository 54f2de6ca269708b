timeout 300 python tools/bias_study.py > gpurun_out/r5_bias.log 2>&1; cat gpurun_out/r5_bias.log
timeout 300 python tools/profile_run.py > gpurun_out/r5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|spmm_onehot" -c 2 -o gpurun_out/r5_prof python tools/profile_run.py > gpurun_out/r5_ncu.log 2>&1
tail -3 gpurun_out/r5_ncu.log
