# round 2: microbenchmarks (TMEM read bandwidth, red.add.u64 throughput); streaming f1 schedule
# variants (block-major BS, supertile raster G); ncu of the supertile variant at n = 200k
mkdir -p gpurun_out
make > gpurun_out/r2_03_make.log 2>&1 || { echo make failed; exit 1; }
./tools/microbench/tmem_ld; ./tools/microbench/red_u64
for v in "KKM_SSYM_BS=16" "KKM_SSYM_BS=8" "KKM_SSYM_G=8" "KKM_SSYM_G=16" "KKM_SSYM_G=32"; do
  echo "== $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --n 200000 --iters 4 --path stream 2>&1 | tail -1 | cut -c150-330
done
for v in "KKM_SSYM_BS=16" "KKM_SSYM_G=16"; do
  echo "== 1M $v"
  env $v timeout 300 python tools/bench_configs.py --configs mnist1m --iters 2 2>&1 | tail -1 | cut -c150-330
done
export KKM_SSYM_G=16
python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_03_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ssym_kernel -c 1 -o gpurun_out/r2_03_ssym python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_03_ncu.log 2>&1; echo "ncu rc=$?"
