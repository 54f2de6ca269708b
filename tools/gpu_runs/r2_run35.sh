# round 2, 2 GPUs: why the peer-memory window setup falls back (KKM_LSA_DEBUG)
mkdir -p gpurun_out
make > gpurun_out/r2_35_make.log 2>&1 || { echo make failed; exit 1; }
KKM_LSA_DEBUG=1 NCCL_DEBUG=WARN timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 tools/trace_phases.py --config mnist60k --iters 4 > gpurun_out/r2_35_trace.log 2>&1; echo "trace rc=$?"; grep -E "kkm rank|NCCL WARN|rror" gpurun_out/r2_35_trace.log | head -20; grep '"rank"' gpurun_out/r2_35_trace.log | cut -c60-400
