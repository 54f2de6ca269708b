# round 2: ssym epilogue without fp64 (int64 fixed point from fp32), relaxed TMEM-empty arrives
mkdir -p gpurun_out
make > gpurun_out/r2_06_make.log 2>&1 || { echo make failed; exit 1; }
KKM_CHAIN_KB=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream and not full and not equals" > gpurun_out/r2_06_pytest.log 2>&1; echo "pytest chain2 rc=$?"; tail -2 gpurun_out/r2_06_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream and not full and not equals" > gpurun_out/r2_06_pytest0.log 2>&1; echo "pytest chain0 rc=$?"; tail -2 gpurun_out/r2_06_pytest0.log
for v in "KKM_CHAIN_KB=0 KKM_SSYM_BS=16" "KKM_CHAIN_KB=2 KKM_SSYM_BS=16" "KKM_CHAIN_KB=3 KKM_SSYM_BS=16" "KKM_CHAIN_KB=4 KKM_SSYM_BS=16"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c150-330
done
for v in "KKM_CHAIN_KB=0 KKM_SSYM_BS=16" "KKM_CHAIN_KB=3 KKM_SSYM_BS=16"; do
  echo "== 1M $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --iters 2 2>&1 | tail -1 | cut -c150-330
done
export KKM_CHAIN_KB=3 KKM_SSYM_BS=16
python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_06_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ssym -c 1 -o gpurun_out/r2_06_ssym python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_06_ncu.log 2>&1; echo "ncu rc=$?"
