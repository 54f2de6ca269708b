# round 2, 2 GPUs: phase timestamps of the distributed a3/a4 (A/B build with globaltimer stamps)
mkdir -p gpurun_out
KKM_LIBKKM=build/libkkm_lsastamps.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29694 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_37_trace.log 2>&1; echo "trace rc=$?"; grep -E "kkm rank" gpurun_out/r2_37_trace.log | tail -6; grep '"rank"' gpurun_out/r2_37_trace.log | cut -c60-460
