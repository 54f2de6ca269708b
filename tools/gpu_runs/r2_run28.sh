# round 2: ncu --set full of update_grid_kernel (config 2, k = 10), summarised on the box (+ top SASS stall lines)
mkdir -p gpurun_out
make > gpurun_out/r2_28_make.log 2>&1 || { echo make failed; exit 1; }
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:update_grid -s 2 -c 1 -o gpurun_out/r2_28_ug python tools/profile_run.py --config mnist60k --iters 4 > gpurun_out/r2_28_run.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r2_28_ug.ncu-rep > gpurun_out/r2_28_ug.txt 2>&1
ncu -i gpurun_out/r2_28_ug.ncu-rep --page details --csv > gpurun_out/r2_28_ug_details.csv 2>/dev/null
ncu -i gpurun_out/r2_28_ug.ncu-rep --page raw --csv > gpurun_out/r2_28_ug_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_28_ug.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_28_ug_src.csv 2>/dev/null
rm -f gpurun_out/r2_28_ug.ncu-rep
head -16 gpurun_out/r2_28_ug.txt
du -sh gpurun_out
