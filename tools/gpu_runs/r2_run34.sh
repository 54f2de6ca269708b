# round 2, 4 GPUs: distributed a3/a4 over NVLink peer memory (NCCL symmetric window; the S
# allreduce fused into the update): config-2 traces with / without (KKM_LSA=0), multi-GPU parity,
# bench at N = 2, 4
mkdir -p gpurun_out
make > gpurun_out/r2_34_make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 tools/trace_phases.py --config mnist60k --iters 8 > gpurun_out/r2_34_trace_lsa.log 2>&1; echo "trace lsa rc=$?"; grep '"rank"' gpurun_out/r2_34_trace_lsa.log | cut -c60-470; grep -i "error\|Traceback" gpurun_out/r2_34_trace_lsa.log | head -5
KKM_LSA=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29682 tools/trace_phases.py --config mnist60k --iters 8 > gpurun_out/r2_34_trace_nccl.log 2>&1; echo "trace nccl rc=$?"; grep '"rank"' gpurun_out/r2_34_trace_nccl.log | head -1 | cut -c60-470
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_34_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_34_pytest.log; grep -E "^E  " gpurun_out/r2_34_pytest.log | head
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2968$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_34_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_34_bench$g.log | cut -c1-200
done
