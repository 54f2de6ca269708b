# a4 fused into the a3 finalize launch (cooperative, grid-wide release of c by the last block):
# GPU tests on 2 GPUs, the multi-GPU equality run, and an A/B of the 1-GPU bench (KKM_NO_FUSED_A4=1 = before)
mkdir -p gpurun_out
make > /dev/null 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r108_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r108_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 tools/run_multi.py > gpurun_out/r108_multi2.log 2>&1; echo "multi rc=$?"; grep -E "MULTI|36001" gpurun_out/r108_multi2.log | cut -c1-220
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export KKM_NO_FUSED_A4=1; else unset KKM_NO_FUSED_A4; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r108_bench_$v.log 2>&1; echo "bench nofuse=$v rc=$?"
  tail -1 gpurun_out/r108_bench_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['phases_ms_per_step'],d['clocks']['sm_mhz'],d['final_J'],d['gpu_launches'])"
done
unset KKM_NO_FUSED_A4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29693 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r108_bench2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/r108_bench2.log | cut -c1-200
