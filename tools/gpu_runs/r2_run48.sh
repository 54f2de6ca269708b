# round 2, 4 GPUs: multi-GPU parity after the IPC path removal and the full streaming kernel's dynamic
# schedule; config 4 1.5D 2x2 vs 1x4 (the full kernel serves 1.5D); bench N = 2, 4
mkdir -p gpurun_out
make > gpurun_out/r2_48_make.log 2>&1 || { echo make failed; exit 1; }
timeout 2400 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_48_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_48_pytest.log; grep -E "^E  " gpurun_out/r2_48_pytest.log | head -5
for gr in 2 1; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2978$gr tools/bench_configs.py --configs mnist1m --iters 5 --grid-rows $gr > gpurun_out/r2_48_mnist1m_g$gr.log 2>&1; echo "mnist1m grid $gr rc=$?"; grep '^{' gpurun_out/r2_48_mnist1m_g$gr.log | cut -c1-420
done
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2979$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_48_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_48_bench$g.log | cut -c1-160
done
