# round 2: multi-GPU (2 GPUs) after the chained-kernel / API refactor: run_multi parity (1D, 1.5D,
# f1 paths, incremental, stop-on-no-change, peer exchange opt-in) and the bench line at N = 2
mkdir -p gpurun_out
make > gpurun_out/r2_11_make.log 2>&1 || { echo make failed; exit 1; }
nvidia-smi -L
timeout 1200 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_11_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_11_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/run_multi.py > gpurun_out/r2_11_multi.log 2>&1; echo "multi rc=$?"; grep -E "MULTI|J\(final\)" gpurun_out/r2_11_multi.log | head; grep -c "labels==oracle True" gpurun_out/r2_11_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2_11_bench2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/r2_11_bench2.log | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/bench_configs.py --configs mnist1m --iters 2 > gpurun_out/r2_11_cfg4_2gpu.log 2>&1; echo "cfg4 2gpu rc=$?"; tail -1 gpurun_out/r2_11_cfg4_2gpu.log | cut -c1-400
