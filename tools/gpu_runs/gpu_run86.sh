python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r86_build.log 2>&1 || { tail -5 gpurun_out/r86_build.log; exit 1; }
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r86_pytest.log 2>&1; tail -2 gpurun_out/r86_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r86_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r86_bench.log').read().strip().split('\n')[-1])
for key in ('value','ms_per_step','clocks','roofline','roofline_a2_phase','e2e','gpu_launches','final_J','cpu_baseline'): print(key, d[key])
PY
