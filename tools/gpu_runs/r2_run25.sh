# round 2: colpart reduction with a bounded, unrolled slab loop (k = 17..32 on 16-bit bands); k = 256 / 900
# parity; config-2-shaped k = 10 / 32 timing; bench line (stream roofline fields)
mkdir -p gpurun_out
make > gpurun_out/r2_25_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -m gpu -x -q -k "32_labels or huge_k or kx2 or many" > gpurun_out/r2_25_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_25_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_25_pytest.log | head
for kk in 10 32; do
  echo "== k=$kk"; timeout 600 python tools/bench_configs.py --configs mnist60k --k $kk --iters 100 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*\|"phases_ms_per_iter": {[^}]*}' | tr '\n' ' '; echo
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:colpart -s 1 -c 1 python tools/profile_run.py --config mnist60k --k 32 --iters 3 > gpurun_out/r2_25_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "duration|dram" gpurun_out/r2_25_ncu.log
timeout 900 python bench.py > gpurun_out/r2_25_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_25_bench.log | cut -c1-200
python - <<'PY'
import json
l = json.loads(open("gpurun_out/r2_25_bench.log").read().strip().splitlines()[-1])
print({k: l.get(k) for k in ("value", "e2e", "clocks", "gpu_launches")})
print(json.dumps(l.get("stream_config4_informational"))[:1200])
PY
