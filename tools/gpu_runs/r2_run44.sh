# round 2, final 4-GPU validation: multi-GPU parity (2, 4, 2 with KKM_LSA=1), bench at N = 2, 4,
# configs 3 and 4 at 2 and 4 GPUs (1D f1), config 4 1.5D 2x2, config 5 at 4 GPUs
mkdir -p gpurun_out
make > gpurun_out/r2_44_make.log 2>&1 || { echo make failed; exit 1; }
timeout 2400 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_44_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_44_pytest.log
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2974$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_44_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_44_bench$g.log | cut -c1-160
done
for g in 2 4; do
  for c in har200k mnist1m; do
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2975$g tools/bench_configs.py --configs $c --iters 5 > gpurun_out/r2_44_${c}_$g.log 2>&1; echo "$c x$g rc=$?"; grep '^{' gpurun_out/r2_44_${c}_$g.log | cut -c1-330
  done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29760 tools/bench_configs.py --configs mnist1m --iters 5 --grid-rows 2 > gpurun_out/r2_44_mnist1m_15d.log 2>&1; echo "mnist1m 2x2 rc=$?"; grep '^{' gpurun_out/r2_44_mnist1m_15d.log | cut -c1-330
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 tools/bench_configs.py --configs mnist8m --iters 2 > gpurun_out/r2_44_mnist8m.log 2>&1; echo "mnist8m x4 rc=$?"; grep '^{' gpurun_out/r2_44_mnist8m.log | cut -c1-330
