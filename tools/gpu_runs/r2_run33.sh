# round 2, 4 GPUs: where the NVLS fused a3/a4's time goes -- A/B build with the cross-rank barrier but
# local S reads (build/libkkm_nvlslocal.so, wrong sums: timing only) vs the real multicast reads
mkdir -p gpurun_out
for lib in "" build/libkkm_nvlslocal.so; do
  KKM_LIBKKM=$lib timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 tools/trace_phases.py --config mnist60k --iters 8 > gpurun_out/r2_33_trace.log 2>&1; echo "trace lib=$lib rc=$?"; grep '"rank"' gpurun_out/r2_33_trace.log | cut -c60-420
done
