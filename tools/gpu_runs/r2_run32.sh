# round 2, 4 GPUs: NVSwitch multicast S exchange fused into the one-launch a3/a4 (setup_nvls,
# multimem.ld_reduce): multi-GPU parity, config-2 traces and bench at N = 2, 4 with and without it
mkdir -p gpurun_out
make > gpurun_out/r2_32_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_32_trace_nvls.log 2>&1; echo "trace nvls rc=$?"; grep '"rank"' gpurun_out/r2_32_trace_nvls.log | cut -c1-500; grep -i "error\|Traceback" gpurun_out/r2_32_trace_nvls.log | head -5
KKM_NVLS=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29662 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_32_trace_nccl.log 2>&1; echo "trace nccl rc=$?"; grep '"rank"' gpurun_out/r2_32_trace_nccl.log | head -1 | cut -c1-500
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_32_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_32_pytest.log
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2967$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_32_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_32_bench$g.log | cut -c1-200
done
