# round 2: full GPU suite + bench (N = 1) after the ssym dynamic schedule / supertile order; ncu --set full
# of ssym at n = 200k and 1M, and of spmm_tc_kernel<32> + its column-partial reduction (config 2, k = 32)
mkdir -p gpurun_out
make > gpurun_out/r2_23_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_23_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_23_pytest.log
timeout 900 python bench.py > gpurun_out/r2_23_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_23_bench.log | cut -c1-300
python - <<'PY'
import json
l = json.loads(open("gpurun_out/r2_23_bench.log").read().strip().splitlines()[-1])
print({k: l.get(k) for k in ("value", "roofline", "clocks", "gpu_launches")})
print(json.dumps(l.get("stream_config4_informational"))[:900])
PY
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:ssym -c 1 -o gpurun_out/r2_23_ssym200k python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_23_ncu1.log 2>&1; echo "ncu ssym200k rc=$?"
timeout 900 ncu $F -k regex:spmm_tc -s 1 -c 1 -o gpurun_out/r2_23_spmmtc32 python tools/profile_run.py --config mnist60k --k 32 --iters 3 > gpurun_out/r2_23_ncu2.log 2>&1; echo "ncu spmm_tc32 rc=$?"
timeout 900 ncu $F -k regex:colpart -s 1 -c 1 -o gpurun_out/r2_23_colpart python tools/profile_run.py --config mnist60k --k 32 --iters 3 > gpurun_out/r2_23_ncu3.log 2>&1; echo "ncu colpart rc=$?"
timeout 900 ncu $F -k regex:spmm_tc -s 1 -c 1 -o gpurun_out/r2_23_spmmtc16 python tools/profile_run.py --config mnist60k --k 16 --iters 3 > gpurun_out/r2_23_ncu4.log 2>&1; echo "ncu spmm_tc16 rc=$?"
timeout 1200 ncu $F -k regex:ssym -c 1 -o gpurun_out/r2_23_ssym1m python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_23_ncu5.log 2>&1; echo "ncu ssym1m rc=$?"
