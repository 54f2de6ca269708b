make -B > /dev/null 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q -k "not multi_gpu" > gpurun_out/r52_pytest.log 2>&1; tail -2 gpurun_out/r52_pytest.log
for it in 10 30; do timeout 300 python tools/profile_run.py --config mnist60k --iters $it 2>&1 | tail -1; done
timeout 300 python tools/profile_run.py --config har200k --iters 20 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r52_bench.log 2>&1; tail -1 gpurun_out/r52_bench.log | cut -c1-120; python -c "
import json; d=json.loads(open('gpurun_out/r52_bench.log').read().strip().split(chr(10))[-1]); print(d['clocks'], d['phases_ms_per_step'])"
