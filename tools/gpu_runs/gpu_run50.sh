mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r50_bench.log 2>&1; tail -1 gpurun_out/r50_bench.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r50_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r50_ncu_bench.log 2>&1; echo "ncu bench exit $?"
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc2_stream_sym -c 1 -o gpurun_out/r50_stream_sym python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > gpurun_out/r50_ncu.log 2>&1; echo "ncu stream exit $?"
