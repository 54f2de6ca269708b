for kn in 0 1 2 3; do
KKM_T2_KNOBS=$kn timeout 300 python tools/profile_run.py --path stream --config mnist1m --n 200000 --iters 2 > gpurun_out/r13_k$kn.log 2>&1; echo "knobs=$kn $(tail -1 gpurun_out/r13_k$kn.log)"
done
timeout 300 python tools/profile_run.py --path mat --iters 5 > gpurun_out/r13_mat.log 2>&1; tail -2 gpurun_out/r13_mat.log
timeout 300 python tools/profile_run.py --path mat --config har200k --n 100000 --iters 5 > gpurun_out/r13_har.log 2>&1; tail -1 gpurun_out/r13_har.log
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
