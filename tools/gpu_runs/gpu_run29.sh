mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 300 python tools/predict_bench.py --config mnist60k --n 200000 --m 200000 --path stream --reps 3 2>&1 | cut -c1-250
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r29_predict200k.csv timeout 600 python tools/predict_bench.py --config mnist60k --n 200000 --m 200000 --path stream --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r29_predict60k_mat.csv timeout 600 python tools/predict_bench.py --config mnist60k --m 60000 --path mat --reps 1 > /dev/null 2>&1
ls -la gpurun_out/
