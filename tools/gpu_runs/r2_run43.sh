# round 2, final 1-GPU validation: full GPU suite, smoke, bench (N = 1, incl. the config-4 streaming
# line), bench --impl reference, ncu launch list of the bench command, configs 1-4 on 1 GPU
mkdir -p gpurun_out
make > gpurun_out/r2_43_make.log 2>&1 || { echo make failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_43_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_43_pytest.log; grep -E "^FAILED|^E  " gpurun_out/r2_43_pytest.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_43_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_43_smoke.log
timeout 1200 python bench.py > gpurun_out/r2_43_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_43_bench.log | cut -c1-160
timeout 1200 python bench.py --impl reference > gpurun_out/r2_43_bench_ref.log 2>&1; echo "bench ref rc=$?"; tail -1 gpurun_out/r2_43_bench_ref.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_43_launches.csv python bench.py --steps 2 --warmup 1 --stream-iters 0 --no-cpu-baseline > gpurun_out/r2_43_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py --launches gpurun_out/r2_43_launches.csv > gpurun_out/r2_43_launches.txt 2>&1; head -12 gpurun_out/r2_43_launches.txt
timeout 1500 python tools/bench_configs.py --configs rings,mnist60k,har200k,mnist1m --iters 5 > gpurun_out/r2_43_configs.log 2>&1; echo "configs rc=$?"; grep '^{' gpurun_out/r2_43_configs.log | cut -c1-330
