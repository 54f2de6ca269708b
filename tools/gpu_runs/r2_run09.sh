# round 2: spmm_tc lo plane first; kx2 / kstore parity; bench with the 1M streaming line
mkdir -p gpurun_out
make > gpurun_out/r2_09_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kstore.py -m gpu -q -k "kx2 or kstore or extreme or large_d or symmetric_bands" > gpurun_out/r2_09_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_09_pytest.log; grep -E "^E  |_ test_" gpurun_out/r2_09_pytest.log | head -10
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_09_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_09_bench.log | python3 -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['value'], l['roofline']['frac'], l['roofline_a1']['frac'], l['clocks']); print(json.dumps(l['stream_config4_informational']))"
