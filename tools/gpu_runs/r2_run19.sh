# round 2: ssym dynamic unit schedule (global counter + smem ring) -- parity subset, then A/B vs the
# static round robin (KKM_SSYM_STATIC) and block-major vs supertile order at 200k / 1M + ncu dram
mkdir -p gpurun_out
make > gpurun_out/r2_19_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "stream or symmetric or large_d" > gpurun_out/r2_19_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_19_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullscale.py -x -q -m gpu -k "config4_recipe" > gpurun_out/r2_19_pytest2.log 2>&1; echo "pytest2 rc=$?"; tail -2 gpurun_out/r2_19_pytest2.log
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | cut -c150-330; }
echo "== dyn BS16 200k"; run "--n 200000" 4
echo "== dyn G16 200k"; KKM_SSYM_G=16 run "--n 200000" 4
echo "== dyn BS16 1M"; run "" 2
echo "== dyn G16 1M"; KKM_SSYM_G=16 run "" 2
echo "== static BS16 1M"; KKM_SSYM_STATIC=1 run "" 2
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_19_ncu_bs.log 2>&1; echo "ncu bs rc=$?"; grep -E "dram__|hit_rate|duration|per_second|inst_exec" gpurun_out/r2_19_ncu_bs.log
KKM_SSYM_G=16 ncu --metrics $M --clock-control none -k regex:ssym -c 1 python tools/profile_run.py --config mnist1m --path stream --iters 1 > gpurun_out/r2_19_ncu_g.log 2>&1; echo "ncu g rc=$?"; grep -E "dram__|hit_rate|duration|per_second|inst_exec" gpurun_out/r2_19_ncu_g.log
