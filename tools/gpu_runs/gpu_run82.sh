make > /dev/null 2>&1 || exit 1
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r82_bench$N.log 2>&1; python - <<PY
import json
d=json.loads(open('gpurun_out/r82_bench$N.log').read().strip().split('\n')[-1])
print($N, d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r82_bench1.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r82_bench1.log').read().strip().split('\n')[-1])
print(1, d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
