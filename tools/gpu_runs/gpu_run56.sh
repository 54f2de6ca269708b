make -B > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r56_bench1.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r56_bench1.log').read().strip().split(chr(10))[-1])
print(d['value'], d['clocks'], d['f3_incremental_informational'])"
timeout 600 python -m pytest tests/test_gpu_kpp.py -q -k quality 2>&1 | tail -1
