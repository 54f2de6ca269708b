# round 2, final 1-GPU run: chain length A/B for the band GEMM (KKM_CHAIN_KB), then the full GPU suite,
# smoke and the bench line on the final build
mkdir -p gpurun_out
make > gpurun_out/r2_50_make.log 2>&1 || { echo make failed; exit 1; }
for ckb in 4 7 13; do
  echo "== KKM_CHAIN_KB=$ckb"; KKM_CHAIN_KB=$ckb timeout 300 python tools/profile_run.py --config mnist60k --iters 2 2>&1 | grep -o "'init_gemm': [0-9.]*"
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_50_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_50_pytest.log; grep -E "^FAILED|^E  " gpurun_out/r2_50_pytest.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_50_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_50_smoke.log
timeout 1200 python bench.py > gpurun_out/r2_50_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_50_bench.log | cut -c1-200
