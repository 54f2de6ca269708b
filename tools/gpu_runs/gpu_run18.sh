timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r18_pytest.log; cat gpurun_out/r18_pytest.log
for k in 10 12 16; do timeout 300 python tools/profile_run.py --path mat --iters 5 --k $k > gpurun_out/r18_k$k.log 2>&1; echo "k=$k $(tail -n 1 gpurun_out/r18_k$k.log)"; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r18_bench.log 2>&1; tail -n 1 gpurun_out/r18_bench.log
timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r18_bench_plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r18_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r18_ncu_launch.log 2>&1; tail -n 2 gpurun_out/r18_ncu_launch.log
