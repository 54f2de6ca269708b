mkdir -p gpurun_out
make -B > /dev/null 2>&1 || exit 1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "rings or edge or empty or symmetric_bands and 3 or incremental and mat and mnist60k-3000" -p no:cacheprovider > gpurun_out/r45_memcheck.log 2>&1; echo "memcheck exit $?"; tail -5 gpurun_out/r45_memcheck.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_predict.py -x -q -k "empty_cluster or training" -p no:cacheprovider > gpurun_out/r45_memcheck2.log 2>&1; echo "memcheck2 exit $?"; tail -3 gpurun_out/r45_memcheck2.log
