for k in 10 8 6 12 16; do timeout 300 python tools/profile_run.py --path mat --iters 5 --k $k > gpurun_out/r17_k$k.log 2>&1; echo "k=$k $(tail -1 gpurun_out/r17_k$k.log)"; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r17_pytest.log; cat gpurun_out/r17_pytest.log
