# round 2: config-5 recipe (n = 8.1M) row-sampled oracle parity on 1 GPU; streaming f1 schedule invariance
mkdir -p gpurun_out
make > gpurun_out/r2_46_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -m gpu -q -x -k "config5 or schedule_invariance" --durations=5 > gpurun_out/r2_46_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r2_46_pytest.log; grep -E "^E  " gpurun_out/r2_46_pytest.log | head
