# round 2, 2 GPUs: peer-memory distributed a3/a4 active -- trace + quick multi-GPU parity (2 ranks)
mkdir -p gpurun_out
make > gpurun_out/r2_36_make.log 2>&1 || { echo make failed; exit 1; }
KKM_LSA_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_36_trace.log 2>&1; echo "trace rc=$?"; grep -E "kkm rank|rror" gpurun_out/r2_36_trace.log | head -8; grep '"rank"' gpurun_out/r2_36_trace.log | cut -c60-460
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29693 tools/run_multi.py > gpurun_out/r2_36_multi.log 2>&1; echo "multi rc=$?"; tail -12 gpurun_out/r2_36_multi.log | cut -c1-300
