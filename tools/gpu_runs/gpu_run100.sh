make > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kstore.py -q -k "stored" 2>&1 | tail -15
