# round 2: ncu --set full of the band GEMM (tc3_gemm_kernel<T2MultiSched>, config 2) with source-level
# stall samples, summarised on the box: is the MMA issuer waiting on the producer (full) or the
# epilogue (cempty)?
mkdir -p gpurun_out
make > gpurun_out/r2_30_make.log 2>&1 || { echo make failed; exit 1; }
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:tc3_gemm -c 1 -o gpurun_out/r2_30_gemm python tools/profile_run.py --config mnist60k --iters 1 > gpurun_out/r2_30_run.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r2_30_gemm.ncu-rep > gpurun_out/r2_30_gemm.txt 2>&1
ncu -i gpurun_out/r2_30_gemm.ncu-rep --page details --csv > gpurun_out/r2_30_gemm_details.csv 2>/dev/null
ncu -i gpurun_out/r2_30_gemm.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_30_gemm_src.csv 2>/dev/null
ncu -i gpurun_out/r2_30_gemm.ncu-rep --page source --csv --print-source cuda > gpurun_out/r2_30_gemm_cu.csv 2>/dev/null
rm -f gpurun_out/r2_30_gemm.ncu-rep
head -16 gpurun_out/r2_30_gemm.txt
du -sh gpurun_out
