T="timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python tools/bench_configs.py --configs rings,mnist60k,har200k --iters 10 > gpurun_out/r19_n1.log 2>&1; grep config gpurun_out/r19_n1.log
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r19_n1b.log 2>&1; grep config gpurun_out/r19_n1b.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29601 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r19_n2.log 2>&1; grep config gpurun_out/r19_n2.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29602 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r19_n2b.log 2>&1; grep config gpurun_out/r19_n2b.log
$T --nproc-per-node 4 --master-port 29603 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r19_n4.log 2>&1; grep config gpurun_out/r19_n4.log
$T --nproc-per-node 4 --master-port 29604 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r19_n4b.log 2>&1; grep config gpurun_out/r19_n4b.log
$T --nproc-per-node 4 --master-port 29605 tools/bench_configs.py --configs mnist1m,har200k --iters 3 --grid-rows 2 > gpurun_out/r19_n4c.log 2>&1; grep config gpurun_out/r19_n4c.log
$T --nproc-per-node 4 --master-port 29606 tools/bench_configs.py --configs mnist8m --iters 1 > gpurun_out/r19_n4d.log 2>&1; grep -E "config|Error" gpurun_out/r19_n4d.log | tail -3
