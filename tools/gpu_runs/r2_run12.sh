# round 2: spmm_tc with 32-label one-hots (16 < k <= 32): parity, then config-2-shaped k = 10 vs 32
mkdir -p gpurun_out
make > gpurun_out/r2_12_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -m gpu -q -x -k "32_labels or many or very or kx2" > gpurun_out/r2_12_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_12_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_12_pytest.log | head
for kk in 10 16 24 32; do
  echo "== k=$kk"; timeout 600 python tools/bench_configs.py --configs mnist60k --k $kk --iters 100 2>&1 | tail -1 | cut -c1-480
done
echo "== k=32 fp32 bands / full K fallback"; timeout 600 python tools/bench_configs.py --configs mnist60k --k 32 --iters 100 --kstore fp32 2>&1 | tail -1 | cut -c1-400
