# round 2, 2 GPUs: distributed a3/a4 with a phase-0 reduce of the own rows' S (stamps build + plain), parity
mkdir -p gpurun_out
make > gpurun_out/r2_38_make.log 2>&1 || { echo make failed; exit 1; }
KKM_LIBKKM=build/libkkm_lsastamps.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29695 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_38_trace_st.log 2>&1; echo "trace stamps rc=$?"; grep -E "kkm rank" gpurun_out/r2_38_trace_st.log | tail -4
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29696 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_38_trace.log 2>&1; echo "trace rc=$?"; grep '"rank"' gpurun_out/r2_38_trace.log | cut -c60-460
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29697 tools/run_multi.py > gpurun_out/r2_38_multi.log 2>&1; echo "multi rc=$?"; tail -3 gpurun_out/r2_38_multi.log | cut -c1-300
