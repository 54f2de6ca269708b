make -B > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r59_bench1.log 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r59_bench1.log').read().strip().split('\n')[-1])
for k in ('value','clocks','roofline','roofline_a2_phase','phases_ms_per_step'): print(k, d[k])
PY
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rings or config2" 2>&1 | tail -1
