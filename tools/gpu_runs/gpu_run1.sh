set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "fp32 or errors" 2>&1 | tail -30 > gpurun_out/r1_pytest.log
cat gpurun_out/r1_pytest.log
timeout 600 python bench.py --precision fp32 --steps 2 --warmup 3 --iters 20 --no-cpu-baseline > gpurun_out/r1_bench.log 2>&1
tail -5 gpurun_out/r1_bench.log
