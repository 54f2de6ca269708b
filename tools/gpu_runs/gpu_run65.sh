make -B > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r65_pytest.log 2>&1; tail -3 gpurun_out/r65_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r65_bench.log 2>&1; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r65_bench.log').read().strip().split('\n')[-1])
print(d['value'], d['clocks'], d['roofline'], d['roofline_a2_phase'], d['phases_ms_per_step'])
PY
timeout 600 ncu --kernel-name regex:spmm_sym --launch-skip 2 --launch-count 1 --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  python tools/profile_run.py --config mnist60k --iters 4 > gpurun_out/r65_ncu.log 2>&1; grep -E "duration|bytes" gpurun_out/r65_ncu.log
