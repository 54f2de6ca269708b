# round 2, 4 GPUs: 1.5D (2x2) vs 1D (1x4) per-iteration phase traces at configs 3 and 4 after the
# send/recv column reduce-scatter (first use vs steady state; a2 - a2_kernel = the exchange), and the
# multi-GPU parity suite
mkdir -p gpurun_out
make > gpurun_out/r2_20_make.log 2>&1 || { echo make failed; exit 1; }
for c in har200k mnist1m; do
  for gr in 1 2; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2961$gr tools/trace_phases.py --config $c --iters 6 --grid-rows $gr > gpurun_out/r2_20_trace_${c}_g$gr.log 2>&1; echo "$c grid $gr rc=$?"; grep '"rank"' gpurun_out/r2_20_trace_${c}_g$gr.log | cut -c1-600
  done
done
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_20_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_20_pytest.log
for c in mnist1m mnist8m; do
  it=5; [ $c = mnist8m ] && it=2
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29620 tools/bench_configs.py --configs $c --iters $it > gpurun_out/r2_20_cfg_$c.log 2>&1; echo "$c 1x4 rc=$?"; tail -1 gpurun_out/r2_20_cfg_$c.log | cut -c1-420
done
