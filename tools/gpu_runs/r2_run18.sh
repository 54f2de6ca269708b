# round 2: epilogue / producer waits with nanosleep backoff; 1M streaming f1: block-major (BS 16) vs
# supertile (G 16) timing + ncu dram / L2 / clock / tensor counters
mkdir -p gpurun_out
make > gpurun_out/r2_18_make.log 2>&1 || { echo make failed; exit 1; }
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | cut -c150-330; }
echo "== BS16 200k"; run "--n 200000" 4
echo "== BS16 1M"; run "" 2
echo "== G16 1M"; KKM_SSYM_G=16 run "" 2
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum
python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_18_plain.log 2>&1
ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_18_ncu_bs.log 2>&1; echo "ncu bs rc=$?"; grep -E "dram__|hit_rate|duration|per_second|tensor|inst_exec" gpurun_out/r2_18_ncu_bs.log
KKM_SSYM_G=16 ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_18_ncu_g.log 2>&1; echo "ncu g rc=$?"; grep -E "dram__|hit_rate|duration|per_second|tensor|inst_exec" gpurun_out/r2_18_ncu_g.log
