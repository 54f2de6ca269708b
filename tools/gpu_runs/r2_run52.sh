# round 2: bench.py end to end after the oracle-thread fix (N = 1 with cpu_baseline, and the reference arm)
mkdir -p gpurun_out
make > gpurun_out/r2_52_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1200 python bench.py > gpurun_out/r2_52_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_52_bench.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['value'], l['cpu_baseline'], l['clocks'], l['stream_config4_informational']['value'])"
timeout 1200 python bench.py --impl reference > gpurun_out/r2_52_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r2_52_ref.log | cut -c1-200
