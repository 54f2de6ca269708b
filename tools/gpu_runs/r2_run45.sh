# round 2: config 3 (HAR 200k) on 1 GPU -- a2 at 5.0 TB/s vs 12.6 ms in round 1: plane order A/B and ncu dram
mkdir -p gpurun_out
for lib in "" build/libkkm_hifirst.so ""; do
  echo "== lib=$lib"; KKM_LIBKKM=$lib timeout 600 python tools/bench_configs.py --configs har200k --iters 5 2>&1 | tail -1 | grep -o '"phases_ms_per_iter": {[^}]*}'
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmm_tc -s 1 -c 1 python tools/profile_run.py --config har200k --iters 2 > gpurun_out/r2_45_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "duration|dram|per_second|hit" gpurun_out/r2_45_ncu.log
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv
