for v in old new old new; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v"; timeout 300 python tools/profile_run.py --config mnist60k --n 200000 --path stream --iters 3 2>&1 | grep -E "stream a1"
done
for v in old new; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 tools/bench_configs.py --configs mnist1m --iters 3 2>/dev/null | grep -v NCCL | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['n_gpus'], round(d['sec_per_iter'],4), d['phases_ms_per_iter'])"
done
