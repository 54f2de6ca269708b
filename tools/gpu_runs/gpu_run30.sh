mkdir -p gpurun_out
make -B > gpurun_out/r30_build.log 2>&1 || { tail -20 gpurun_out/r30_build.log; exit 1; }
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r30_pytest.log 2>&1; tail -2 gpurun_out/r30_pytest.log
for args in "--config mnist60k --m 60000 --path mat" "--config mnist60k --m 60000 --path stream" "--config mnist60k --n 200000 --m 200000 --path stream" "--config har200k --m 50000 --k 40"; do
  timeout 300 python tools/predict_bench.py $args --reps 3 2>&1 | cut -c1-330; done > gpurun_out/r30_predict.log; cat gpurun_out/r30_predict.log
$T --nproc-per-node 4 --master-port 29711 tools/trace_phases.py --config mnist60k --grid-rows 2 > gpurun_out/r30_trace_m2x2.log 2>&1; cut -c1-400 gpurun_out/r30_trace_m2x2.log | grep config
$T --nproc-per-node 4 --master-port 29712 tools/trace_phases.py --config mnist60k > gpurun_out/r30_trace_m1x4.log 2>&1; cut -c1-400 gpurun_out/r30_trace_m1x4.log | grep config
$T --nproc-per-node 4 --master-port 29713 tools/trace_phases.py --config har200k --grid-rows 2 > gpurun_out/r30_trace_h2x2.log 2>&1; cut -c1-400 gpurun_out/r30_trace_h2x2.log | grep config
