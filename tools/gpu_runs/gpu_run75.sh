make > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r75_launches.csv python tools/profile_run.py --config mnist60k --iters 5 --kstore fp16x2 > gpurun_out/r75.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/r75_launches.csv | head -20
