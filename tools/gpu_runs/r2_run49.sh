# round 2: band GEMM epilogue with two staging slots per warp (column constants read from global):
# parity (materialised paths) and init_gemm A/B against the previous build (build/libkkm_gemmold.so)
mkdir -p gpurun_out
make > gpurun_out/r2_49_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -m gpu -x -q > gpurun_out/r2_49_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_49_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_49_pytest.log | head
for lib in "" build/libkkm_gemmold.so "" build/libkkm_gemmold.so; do
  echo "== lib=$lib"; KKM_LIBKKM=$lib timeout 300 python tools/profile_run.py --config mnist60k --iters 2 2>&1 | grep -o "'init_gemm': [0-9.]*"
done
echo "== har200k (Gaussian) init_gemm"; timeout 300 python tools/profile_run.py --config har200k --n 60000 --iters 2 2>&1 | grep -o "'init_gemm': [0-9.]*"
KKM_LIBKKM=build/libkkm_gemmold.so timeout 300 python tools/profile_run.py --config har200k --n 60000 --iters 2 2>&1 | grep -o "'init_gemm': [0-9.]*"
