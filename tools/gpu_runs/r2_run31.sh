# round 2, 4 GPUs: NCCL collective floor at config-2 sizes (2 and 4 ranks), NCCL_DEBUG for NVLS use
mkdir -p gpurun_out
for g in 2 4; do
  NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2965$g tools/nccl_probe.py > gpurun_out/r2_31_probe$g.log 2>&1; echo "probe$g rc=$?"; grep '^{' gpurun_out/r2_31_probe$g.log
  grep -i "nvls\|algo" gpurun_out/r2_31_probe$g.log | head -5
done
