# round 2: chained accumulation in the streaming f1 kernel (ssym_chain_kernel, KKM_CHAIN_KB) -- parity + speed
mkdir -p gpurun_out
make > gpurun_out/r2_05_make.log 2>&1 || { echo make failed; exit 1; }
for c in 2 1 3; do
KKM_CHAIN_KB=$c timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream and not full" > gpurun_out/r2_05_pytest_c$c.log 2>&1; echo "pytest chain $c rc=$?"; tail -2 gpurun_out/r2_05_pytest_c$c.log
done
for v in "KKM_CHAIN_KB=0 KKM_SSYM_BS=16" "KKM_CHAIN_KB=2 KKM_SSYM_BS=16" "KKM_CHAIN_KB=1 KKM_SSYM_BS=16" "KKM_CHAIN_KB=3 KKM_SSYM_BS=16" "KKM_CHAIN_KB=2 KKM_SSYM_G=16" "KKM_CHAIN_KB=2 KKM_SSYM_BS=8"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c150-330
done
for v in "KKM_CHAIN_KB=2 KKM_SSYM_BS=16" "KKM_CHAIN_KB=2 KKM_SSYM_BS=8"; do
  echo "== 1M $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --iters 2 2>&1 | tail -1 | cut -c150-330
done
