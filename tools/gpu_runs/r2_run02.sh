# round 2: the new streaming f1 kernel (ssym.cuh) -- parity, then A/B against the round-1 kernel
mkdir -p gpurun_out
make > gpurun_out/r2_02_make.log 2>&1 || { echo make failed; tail gpurun_out/r2_02_make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream or symmetric or many or very or edge or empty or rings" > gpurun_out/r2_02_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_02_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -x -k "config4" > gpurun_out/r2_02_pytest_fs.log 2>&1; echo "pytest fs rc=$?"; tail -3 gpurun_out/r2_02_pytest_fs.log
for v in "KKM_SSYM_V1=1" "KKM_SSYM_BS=32" "KKM_SSYM_BS=64" "KKM_SSYM_BS=16" "KKM_SSYM_BS=32 KKM_SSYM_TILE_MAJOR=1"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c1-420
done
for v in "KKM_SSYM_V1=1" "KKM_SSYM_BS=32"; do
  echo "== 1M $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --iters 2 2>&1 | tail -1 | cut -c1-420
done
