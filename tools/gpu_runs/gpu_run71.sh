make > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_kstore.py -x -q > gpurun_out/r71_pytest.log 2>&1; tail -3 gpurun_out/r71_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 --kstore fp16 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config har200k --iters 10 --kstore fp16 2>&1 | tail -2
timeout 300 python tools/profile_run.py --config har200k --iters 10 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r71_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r71_bench.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks'], d['roofline']['frac'], d['f4_fp16_kstore_informational'])
PY
