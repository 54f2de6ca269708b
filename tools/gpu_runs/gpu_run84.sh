make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore or symmetric" > gpurun_out/r84_pytest.log 2>&1; tail -1 gpurun_out/r84_pytest.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/run_multi.py > gpurun_out/r84_multi$N.log 2>&1; grep -E "MULTI|False" gpurun_out/r84_multi$N.log | head -5
done
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r84_bench$N.log 2>&1; python - <<PY
import json
d=json.loads(open('gpurun_out/r84_bench$N.log').read().strip().split('\n')[-1])
print($N, d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['final_J'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
done
