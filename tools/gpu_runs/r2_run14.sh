# round 2, 4 GPUs: multi-GPU parity (2 and 4 ranks), bench at N = 1, 2, 4, configs 3 and 4 at 4 GPUs
# (1D f1 vs the 1.5D 2x2 grid), config 5 (n = 8.1M) at 4 GPUs
mkdir -p gpurun_out
make > gpurun_out/r2_14_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_14_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_14_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --stream-iters 0 --no-cpu-baseline > gpurun_out/r2_14_bench1.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/r2_14_bench1.log | cut -c1-130
for g in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2952$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_14_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_14_bench$g.log | cut -c1-130
done
for c in har200k mnist1m; do
  for gr in 1 2; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$gr tools/bench_configs.py --configs $c --iters 5 --grid-rows $gr > gpurun_out/r2_14_${c}_g$gr.log 2>&1; echo "$c grid $gr rc=$?"; tail -1 gpurun_out/r2_14_${c}_g$gr.log | cut -c1-420
  done
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29540 tools/bench_configs.py --configs mnist8m --iters 2 > gpurun_out/r2_14_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -1 gpurun_out/r2_14_cfg5.log | cut -c1-420
