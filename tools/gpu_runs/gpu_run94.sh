make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -x -q -k "kx2 or kstore or symmetric or full_size" > gpurun_out/r94_pytest.log 2>&1; tail -1 gpurun_out/r94_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r94_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r94_bench.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks']['sm_mhz'], d['final_J'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 tools/run_multi.py > gpurun_out/r94_multi2.log 2>&1; grep -E "MULTI" gpurun_out/r94_multi2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r94_bench2.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r94_bench2.log').read().strip().split('\n')[-1])
print(2, d['value'], d['clocks']['sm_mhz'], d['final_J'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
