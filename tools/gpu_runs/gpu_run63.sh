make -B > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r63_pytest.log 2>&1; tail -1 gpurun_out/r63_pytest.log
timeout 300 python tools/profile_run.py --config mnist60k --iters 20 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r63_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r63_bench.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['roofline']['launch_ms'], d['phases_ms_per_step']['a2_kernel'])
PY
