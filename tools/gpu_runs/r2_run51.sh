# round 2: accumulation chains of 7 K-blocks (KKM_CHAIN_KB=7) instead of 4 -- the precision side:
# full-size J against the oracle (configs 1-3), the d = 3000 bias test and the parity suite, vs CKB 4
mkdir -p gpurun_out
make > gpurun_out/r2_51_make.log 2>&1 || { echo make failed; exit 1; }
for ckb in 4 7; do
  KKM_CHAIN_KB=$ckb timeout 1800 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_parity.py -m gpu -q -s -k "objective or large_d or teacher or symmetric" > gpurun_out/r2_51_ckb$ckb.log 2>&1; echo "ckb $ckb rc=$?"; tail -1 gpurun_out/r2_51_ckb$ckb.log; grep -E "J .* oracle .* rel" gpurun_out/r2_51_ckb$ckb.log; grep -E "^E  |^FAILED" gpurun_out/r2_51_ckb$ckb.log | head -5
done
for ckb in 4 7; do
  echo "== ssym 200k KKM_CHAIN_KB=$ckb"; KKM_CHAIN_KB=$ckb timeout 600 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 3 --path stream 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*'
done
