set -x
mkdir -p gpurun_out
make -B > gpurun_out/r28_build.log 2>&1 || { tail -20 gpurun_out/r28_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r28_pytest.log 2>&1; tail -5 gpurun_out/r28_pytest.log
timeout 300 python tools/predict_bench.py --config mnist60k --m 60000 --path mat > gpurun_out/r28_predict.log 2>&1
timeout 300 python tools/predict_bench.py --config mnist60k --m 60000 --path stream >> gpurun_out/r28_predict.log 2>&1
timeout 300 python tools/predict_bench.py --config mnist60k --n 200000 --m 200000 --path stream >> gpurun_out/r28_predict.log 2>&1
timeout 300 python tools/predict_bench.py --config har200k --m 50000 --k 40 >> gpurun_out/r28_predict.log 2>&1
cat gpurun_out/r28_predict.log | cut -c1-400
for k in 10 21 70; do timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --iters 2 --path stream --k $k 2>&1 | tail -1; done > gpurun_out/r28_streamk.log; cat gpurun_out/r28_streamk.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r28_bench.log 2>&1; tail -1 gpurun_out/r28_bench.log | cut -c1-300
