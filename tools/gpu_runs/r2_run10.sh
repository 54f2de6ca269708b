# round 2: validation of the refactored API + chained kernels: GPU suite, smoke, bench; ncu of the
# streaming f1 kernel (n = 200k), of the a1 GEMM (config 2) and the bench's launch list
mkdir -p gpurun_out
make > gpurun_out/r2_10_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/r2_10_pytest.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/r2_10_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_10_pytest.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_10_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_10_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_10_bench.log 2>&1; echo "bench rc=$?"
python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_10_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ssym -c 1 -o gpurun_out/r2_10_ssym python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_10_ncu1.log 2>&1; echo "ncu ssym rc=$?"
python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r2_10_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc3_gemm -c 1 -o gpurun_out/r2_10_gemm python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r2_10_ncu2.log 2>&1; echo "ncu gemm rc=$?"
python bench.py --steps 1 --warmup 3 --stream-iters 0 --no-cpu-baseline > gpurun_out/r2_10_plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_10_launches.csv python bench.py --steps 1 --warmup 3 --stream-iters 0 --no-cpu-baseline > gpurun_out/r2_10_ncu3.log 2>&1; echo "ncu launches rc=$?"
