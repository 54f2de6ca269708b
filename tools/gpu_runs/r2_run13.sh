# round 2: compute-sanitizer memcheck over every hot kernel family (tools/sanitize_run.py), one tool
mkdir -p gpurun_out
make > gpurun_out/r2_13_make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python tools/sanitize_run.py > gpurun_out/r2_13_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2_13_plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2_13_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -8 gpurun_out/r2_13_memcheck.log
