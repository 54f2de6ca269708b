# round 2: L2 promotion of the streaming operand loads (KKM_TS_PROMO); DRAM traffic of ssym at a
# size whose operands fit L2 (n = 20k) vs 200k, with ncu's dram counters only
mkdir -p gpurun_out
make > gpurun_out/r2_17_make.log 2>&1 || { echo make failed; exit 1; }
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | cut -c150-260; }
for pr in 256 128 0; do echo "== promo $pr 200k"; KKM_TS_PROMO=$pr run "--n 200000" 4; done
for pr in 256 128; do echo "== promo $pr 1M"; KKM_TS_PROMO=$pr run "" 2; done
python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_17_plain.log 2>&1
for pr in 256 128; do
KKM_TS_PROMO=$pr ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --n 200000 --path stream --iters 1 > gpurun_out/r2_17_ncu_$pr.log 2>&1; echo "ncu $pr rc=$?"; grep -E "dram__bytes|hit_rate|duration|per_second" gpurun_out/r2_17_ncu_$pr.log
done
KKM_TS_PROMO=256 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --n 20000 --path stream --iters 1 > gpurun_out/r2_17_ncu_20k.log 2>&1; echo "ncu 20k rc=$?"; grep -E "dram__bytes|hit_rate|duration" gpurun_out/r2_17_ncu_20k.log
