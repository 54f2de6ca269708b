for k in 12 16 10; do timeout 300 python tools/profile_run.py --path mat --iters 5 --k $k > gpurun_out/r26_k$k.log 2>&1; echo "k=$k $(tail -n 1 gpurun_out/r26_k$k.log)"; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r26_bench.log 2>&1; tail -n 1 gpurun_out/r26_bench.log | cut -c1-600
