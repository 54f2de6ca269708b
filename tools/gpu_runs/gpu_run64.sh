make -B > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "extreme or large_d" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
