# round 2, 4 GPUs: distributed a3/a4 (phase-0 reduce over all co-resident blocks): stamps, traces,
# multi-GPU parity, bench N = 2, 4 with and without it (KKM_LSA=0)
mkdir -p gpurun_out
make > gpurun_out/r2_39_make.log 2>&1 || { echo make failed; exit 1; }
KKM_LIBKKM=build/libkkm_lsastamps.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_39_trace_st.log 2>&1; echo "trace stamps rc=$?"; grep -E "kkm rank" gpurun_out/r2_39_trace_st.log | tail -4
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_39_trace.log 2>&1; echo "trace rc=$?"; grep '"rank"' gpurun_out/r2_39_trace.log | cut -c60-460
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_39_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_39_pytest.log; grep -E "^E  " gpurun_out/r2_39_pytest.log | head
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2970$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_39_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_39_bench$g.log | cut -c1-150
  KKM_LSA=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2971$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_39_bench${g}_nccl.log 2>&1; echo "bench$g nccl rc=$?"; tail -1 gpurun_out/r2_39_bench${g}_nccl.log | cut -c1-150
done
