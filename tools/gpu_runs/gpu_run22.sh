timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for k in 10 8 6 2 12; do timeout 300 python tools/profile_run.py --path mat --iters 5 --k $k > gpurun_out/r22_k$k.log 2>&1; echo "k=$k $(tail -n 1 gpurun_out/r22_k$k.log)"; done
