for v in s16 s8 s4; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | grep "a2 SpMM"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r85_bench4_$v.log 2>&1; python - <<PY
import json
d=json.loads(open('gpurun_out/r85_bench4_$v.log').read().strip().split('\n')[-1])
print(4, d['value'], d['clocks']['sm_mhz'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
done
