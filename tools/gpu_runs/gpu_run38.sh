mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc2_stream_sym -c 1 -o gpurun_out/r39_stream_sym timeout 600 python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > gpurun_out/r39_ncu.log 2>&1; tail -1 gpurun_out/r39_ncu.log
