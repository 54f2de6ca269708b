# round 2: ssym supertile G32 x W16 at 200k; A/B experiment builds at 1M (build/libkkm_nocol.so:
# column-part atomics removed; build/libkkm_noepi.so: no epilogue arithmetic) -> where the power goes
mkdir -p gpurun_out
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*'; }
echo "== BS16 200k"; run "--n 200000" 4
echo "== G32W16 200k"; KKM_SSYM_G=32 KKM_SSYM_W=16 run "--n 200000" 4
echo "== G32W16 1M"; KKM_SSYM_G=32 KKM_SSYM_W=16 run "" 2
echo "== G32W16 1M nocol"; KKM_LIBKKM=build/libkkm_nocol.so KKM_SSYM_G=32 KKM_SSYM_W=16 run "" 2
echo "== G32W16 1M noepi"; KKM_LIBKKM=build/libkkm_noepi.so KKM_SSYM_G=32 KKM_SSYM_W=16 run "" 2
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum
for v in nocol noepi; do
KKM_LIBKKM=build/libkkm_$v.so KKM_SSYM_G=32 KKM_SSYM_W=16 ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_22_ncu_$v.log 2>&1; echo "ncu $v rc=$?"; grep -E "dram__|hit_rate|duration|per_second|inst_exec" gpurun_out/r2_22_ncu_$v.log
done
