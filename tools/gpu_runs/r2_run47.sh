# round 2: the full streaming kernel on W-column units in G-row supertiles, taken dynamically (the
# ssym ring moved into chain.cuh): streaming parity (full kernel, predict, incremental, 300k sampled),
# config-4 recipe with the full kernel (SYM_OFF) at 200k / 1M: dynamic vs round 1's long static units
mkdir -p gpurun_out
make > gpurun_out/r2_47_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_predict.py tests/test_gpu_fullscale.py -m gpu -x -q -k "stream or predict or incremental or 300k or config4 or schedule" > gpurun_out/r2_47_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_47_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_47_pytest.log | head
run() { timeout 900 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream --symmetric off 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*\|"a2_kernel": [0-9.]*' | tr '\n' ' '; echo; }
echo "== 200k dyn G32 W16"; run "--n 200000" 3
echo "== 200k static long units"; KKM_SSYM_STATIC=1 KKM_TS_G=1 KKM_TS_W=512 run "--n 200000" 3
echo "== 1M dyn G32 W16"; run "" 2
echo "== 1M static long units"; KKM_SSYM_STATIC=1 KKM_TS_G=1 KKM_TS_W=512 run "" 2
echo "== predict 200k x 200k"; timeout 600 python tools/predict_bench.py --config mnist1m --n 200000 --m 200000 --path stream --reps 3 2>&1 | tail -1 | cut -c1-300
echo "== predict 200k x 200k static long"; KKM_SSYM_STATIC=1 KKM_TS_G=1 KKM_TS_W=512 timeout 600 python tools/predict_bench.py --config mnist1m --n 200000 --m 200000 --path stream --reps 3 2>&1 | tail -1 | cut -c1-300
