# round 2: ssym dynamic schedule, unit shape / order sweep at n = 1M (block-major BS; supertile G with
# W column tiles per unit) + ncu dram / clock of the best candidates
mkdir -p gpurun_out
make > gpurun_out/r2_21_make.log 2>&1 || { echo make failed; exit 1; }
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | grep -o '"sec_per_iter": [0-9.]*'; }
echo "== BS16"; run "" 2
echo "== BS32"; KKM_SSYM_BS=32 run "" 2
echo "== G16 W4"; KKM_SSYM_G=16 KKM_SSYM_W=4 run "" 2
echo "== G16 W8"; KKM_SSYM_G=16 KKM_SSYM_W=8 run "" 2
echo "== G32 W8"; KKM_SSYM_G=32 KKM_SSYM_W=8 run "" 2
echo "== G32 W16"; KKM_SSYM_G=32 KKM_SSYM_W=16 run "" 2
echo "== G64 W16"; KKM_SSYM_G=64 KKM_SSYM_W=16 run "" 2
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum
for v in "16 4" "32 8" "32 16"; do set -- $v
KKM_SSYM_G=$1 KKM_SSYM_W=$2 ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_21_ncu_g$1w$2.log 2>&1; echo "ncu G$1 W$2 rc=$?"; grep -E "dram__|hit_rate|duration|per_second|inst_exec" gpurun_out/r2_21_ncu_g$1w$2.log
done
