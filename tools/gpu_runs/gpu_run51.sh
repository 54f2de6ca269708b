make -B > /dev/null 2>&1 || exit 1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 tools/run_multi.py > gpurun_out/r51_multi.log 2>&1; echo "exit $?"
grep -E "P=2|MULTI" gpurun_out/r51_multi.log | cut -c1-230
