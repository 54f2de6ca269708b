# round 2, 4 GPUs: NCCL allreduce of S on an NCCL symmetric window (KKM_LSA=2) vs plain device memory
mkdir -p gpurun_out
make > gpurun_out/r2_42_make.log 2>&1 || { echo make failed; exit 1; }
for v in 0 2; do
  KKM_LSA=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2972$v tools/trace_phases.py --config mnist60k --iters 8 > gpurun_out/r2_42_trace$v.log 2>&1; echo "trace KKM_LSA=$v rc=$?"; grep '"rank"' gpurun_out/r2_42_trace$v.log | head -2 | cut -c60-470
done
