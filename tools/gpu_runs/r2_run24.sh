# round 2: GEMM supertile order (KKM_GEMM_GR) A/B + parity; ncu --set full of ssym (200k, 1M), spmm_tc<32>,
# spmm_tc<16>, the column-partial reduction and the band GEMM, summarised ON the box (reports deleted:
# the merge-back limit is 64 MiB)
mkdir -p gpurun_out
make > gpurun_out/r2_24_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -m gpu -x -q > gpurun_out/r2_24_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_24_pytest.log
for gr in 0 32 16 64; do
  echo "== GEMM_GR=$gr"; KKM_GEMM_GR=$gr timeout 600 python tools/bench_configs.py --configs mnist60k --iters 20 2>&1 | tail -1 | grep -o '"init_s": [0-9.]*\|"sec_per_iter": [0-9.]*\|"init_gemm_ms": [0-9.]*\|"a1_roofline": {[^}]*}' | tr '\n' ' '; echo
done
F="--set full --clock-control none --import-source on"
S=tools/ncu_summary.py
prof() {  # name, kernel regex, launch skip, profile_run args...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 1200 ncu $F -k regex:$kre -s $skip -c 1 -o gpurun_out/$name python tools/profile_run.py "$@" > gpurun_out/${name}_run.log 2>&1; echo "ncu $name rc=$?"
  python $S gpurun_out/$name.ncu-rep > gpurun_out/$name.txt 2>&1
  ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_src.csv 2>/dev/null
  gzip -f gpurun_out/${name}_src.csv
  rm -f gpurun_out/$name.ncu-rep
  head -16 gpurun_out/$name.txt
}
prof r2_24_gemm tc3_gemm 1 --config mnist60k --iters 1
prof r2_24_ssym200k ssym 0 --config mnist1m --n 200000 --path stream --iters 1
prof r2_24_spmmtc32 spmm_tc 1 --config mnist60k --k 32 --iters 3
prof r2_24_spmmtc16 spmm_tc 1 --config mnist60k --k 16 --iters 3
prof r2_24_colpart colpart 1 --config mnist60k --k 32 --iters 3
prof r2_24_ssym1m ssym 0 --config mnist1m --path stream --iters 1
du -sh gpurun_out
