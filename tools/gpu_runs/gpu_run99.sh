timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r99_bench1.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r99_bench1.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['fp32_bands_informational'], d['f4_fp16_kstore_informational']['total_clustering_s'])
PY
