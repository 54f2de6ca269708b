make -B > /dev/null 2>&1 || exit 1
timeout 600 python tools/j_precision.py --config mnist60k 2>&1 | tail -1
timeout 600 python tools/j_precision.py --config mnist60k --symmetric off 2>&1 | tail -1
timeout 900 python tools/j_precision.py --config har200k --iters 30 2>&1 | tail -1
timeout 600 python tools/j_precision.py --config rings 2>&1 | tail -1
