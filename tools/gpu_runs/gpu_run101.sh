make > /dev/null 2>&1 || exit 1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/run_multi.py > gpurun_out/r101_multi2.log 2>&1; echo "rc=$?"; grep -E "MULTI|kstore|symmetric" gpurun_out/r101_multi2.log | cut -c1-200; tail -3 gpurun_out/r101_multi2.log | cut -c1-300
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r101_bench$N.log 2>&1; echo "rc=$?"; python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/r101_bench$N.log').read().strip().split('\n') if l.startswith('{')][-1])
print($N, d['value'], d['clocks']['sm_mhz'], d['final_J'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
done
