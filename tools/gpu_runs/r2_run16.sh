# round 2: L2 policy of the streaming f1 kernel's operand loads (KKM_SSYM_HINT) and block size at 1M
mkdir -p gpurun_out
make > gpurun_out/r2_16_make.log 2>&1 || { echo make failed; exit 1; }
run() { timeout 600 python tools/bench_configs.py --configs mnist1m $1 --iters $2 --path stream 2>&1 | tail -1 | cut -c150-260; }
for hnt in 1 0 2 3 4; do echo "== hint $hnt 200k"; KKM_SSYM_HINT=$hnt run "--n 200000" 4; done
for hnt in 1 0 2; do echo "== hint $hnt 1M"; KKM_SSYM_HINT=$hnt run "" 2; done
echo "== hint 1 1M BS8"; KKM_SSYM_BS=8 run "" 2
echo "== hint 0 1M BS8"; KKM_SSYM_HINT=0 KKM_SSYM_BS=8 run "" 2
