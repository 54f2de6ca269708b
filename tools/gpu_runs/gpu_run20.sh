timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream" 2>&1 | tail -1
for kn in 0 2; do KKM_T2_KNOBS=$kn timeout 300 python tools/profile_run.py --path stream --config mnist1m --iters 1 > gpurun_out/r20_k$kn.log 2>&1; echo "knobs=$kn $(tail -n 1 gpurun_out/r20_k$kn.log)"; done
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 2 > gpurun_out/r20_200k.log 2>&1; tail -n 1 gpurun_out/r20_200k.log
