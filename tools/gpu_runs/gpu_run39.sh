mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc2_stream_sym -c 1 -o gpurun_out/r39_stream_sym timeout 600 python tools/profile_run.py --config mnist60k --n 200000 --iters 1 --path stream > gpurun_out/r39_ncu.log 2>&1; tail -1 gpurun_out/r39_ncu.log
python tools/ncu_summary.py gpurun_out/r39_stream_sym.ncu-rep 2>&1 | grep -E "duration|dram__bytes_read|hit_rate|tensor_cycles"
for a in "" "--full-k"; do timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 3 --path stream $a 2>&1 | tail -1; done
timeout 300 python tools/profile_run.py --config har200k --iters 3 --path stream 2>&1 | tail -1
timeout 600 python tools/profile_run.py --config mnist1m --iters 2 --path stream 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream" 2>&1 | tail -1
