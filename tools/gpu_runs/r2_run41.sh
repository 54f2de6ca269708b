# round 2: band GEMM direct stores vs TMA-staged stores (A/B build), init_gemm phase via profile_run (3 runs each)
mkdir -p gpurun_out
for lib in "" build/libkkm_tmastore.so "" build/libkkm_tmastore.so; do
  echo "== lib=$lib"; KKM_LIBKKM=$lib timeout 300 python tools/profile_run.py --config mnist60k --iters 2 2>&1 | grep -o "'init_gemm': [0-9.]*"
done
