make > /dev/null 2>&1 || exit 1
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$N tools/run_multi.py > gpurun_out/r105_multi$N.log 2>&1; echo "rc=$?"; grep -E "MULTI|36001" gpurun_out/r105_multi$N.log | cut -c1-220
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29699 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r105_bench4.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/r105_bench4.log | cut -c1-110
