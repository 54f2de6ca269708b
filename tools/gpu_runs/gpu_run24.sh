for k in 10 6; do timeout 300 python tools/profile_run.py --path mat --iters 5 --k $k > gpurun_out/r24_k$k.log 2>&1; echo "k=$k $(tail -n 1 gpurun_out/r24_k$k.log)"; done
timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 2 > gpurun_out/r24_s.log 2>&1; tail -n 1 gpurun_out/r24_s.log
timeout 300 python tools/profile_run.py --path stream --config mnist1m --iters 1 > gpurun_out/r24_s1m.log 2>&1; tail -n 1 gpurun_out/r24_s1m.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
