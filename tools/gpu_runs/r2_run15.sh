# round 2: mbarrier waits with a suspend-time hint (A/B against gpurun_vars/libkkm_nohint.so) on the
# streaming f1 kernel at n = 200k and 1M; unit raster (block 16 vs supertile 16); ncu at 1M
mkdir -p gpurun_out
make > gpurun_out/r2_15_make.log 2>&1 || { echo make failed; exit 1; }
cp paper_2601_17136_b200/libkkm.so gpurun_vars/libkkm_hint.so
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | cut -c150-300; }
for v in nohint hint nohint hint; do
  cp gpurun_vars/libkkm_$v.so paper_2601_17136_b200/libkkm.so
  echo "== $v 200k"; run "--n 200000" 4
done
cp gpurun_vars/libkkm_hint.so paper_2601_17136_b200/libkkm.so
echo "== hint 1M BS16"; run "" 2
echo "== hint 1M G16"; KKM_SSYM_G=16 run "" 2
cp gpurun_vars/libkkm_nohint.so paper_2601_17136_b200/libkkm.so
echo "== nohint 1M BS16"; run "" 2
cp gpurun_vars/libkkm_hint.so paper_2601_17136_b200/libkkm.so
python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_15_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ssym -c 1 -o gpurun_out/r2_15_ssym1m python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_15_ncu.log 2>&1; echo "ncu rc=$?"
