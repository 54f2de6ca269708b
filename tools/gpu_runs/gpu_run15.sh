timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r15_pytest.log; cat gpurun_out/r15_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r15_bench.log 2>&1; tail -1 gpurun_out/r15_bench.log
timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r15_bench_plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r15_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r15_ncu_launch.log 2>&1; tail -2 gpurun_out/r15_ncu_launch.log
