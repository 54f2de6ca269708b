# round 2: Gaussian norms from the tensor core's own self dots (A9); full GPU suite; J precision at configs 1-3
mkdir -p gpurun_out
make > gpurun_out/r2_04_make.log 2>&1 || { echo make failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=8 --deselect tests/test_gpu_fullscale.py::test_full_size_objective_at_convergence > gpurun_out/r2_04_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_04_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k objective > gpurun_out/r2_04_jprec.log 2>&1; echo "jprec rc=$?"; grep -E "rel|passed|failed" gpurun_out/r2_04_jprec.log
timeout 300 python tools/bench_configs.py --configs har200k --iters 30 2>&1 | tail -1 | cut -c1-400
