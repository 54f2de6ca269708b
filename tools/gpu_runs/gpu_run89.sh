for v in f0 f1 f0 f1; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r89_bench4_$v.log 2>&1; python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/r89_bench4_$v.log').read().strip().split('\n') if l.startswith('{')][-1])
print('$v', d['value'], d['clocks']['sm_mhz'], {k: round(v/100,4) for k,v in d['phases_ms_per_step'].items()})
PY
done
grep -m3 -i "nvls" gpurun_out/r89_bench4_f1.log
