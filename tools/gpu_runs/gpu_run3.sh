timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "edge and fp32" 2>&1 | head -120 > gpurun_out/r3_edge.log
