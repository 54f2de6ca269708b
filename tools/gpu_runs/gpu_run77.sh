make > /dev/null 2>&1 || exit 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/run_multi.py > gpurun_out/r77_multi.log 2>&1; tail -25 gpurun_out/r77_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r77_bench2.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r77_bench2.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks'], d['roofline']['frac'], d['final_J'], d['phases_ms_per_step'])
PY
