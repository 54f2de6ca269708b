# round 2, 4 GPUs: multi-GPU parity after the one-launch a3/a4 and the ssym dynamic schedule; bench at
# N = 2, 4 (config 2); config-2 per-phase traces at 1x4 (where the fixed per-iteration cost goes)
mkdir -p gpurun_out
make > gpurun_out/r2_29_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1800 python -m pytest tests/test_multi_gpu.py -m gpu -q -rs > gpurun_out/r2_29_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_29_pytest.log
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2963$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_29_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_29_bench$g.log | cut -c1-200
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/trace_phases.py --config mnist60k --iters 6 > gpurun_out/r2_29_trace_c2.log 2>&1; echo "trace rc=$?"; grep '"rank"' gpurun_out/r2_29_trace_c2.log | cut -c1-500
