make > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r76_pytest.log 2>&1; tail -3 gpurun_out/r76_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r76_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r76_bench.log').read().strip().split('\n')[-1])
for key in ('value','clocks','roofline','roofline_a2_phase','phases_ms_per_step','final_J','f4_fp16_kstore_informational'): print(key, d[key])
PY
timeout 900 python bench.py --steps 3 --warmup 3 --kstore fp32 --no-cpu-baseline > gpurun_out/r76_bench_fp32.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r76_bench_fp32.log').read().strip().split('\n')[-1])
print('fp32 bands', d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['final_J'])
PY
