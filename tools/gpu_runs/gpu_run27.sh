T="timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multi_gpu.py -q 2>&1 | tail -1
timeout 900 python tools/bench_configs.py --configs rings,mnist60k,har200k --iters 10 > gpurun_out/r27_n1.log 2>&1; grep config gpurun_out/r27_n1.log
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r27_n1b.log 2>&1; grep config gpurun_out/r27_n1b.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29701 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r27_n2.log 2>&1; grep config gpurun_out/r27_n2.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29702 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r27_n2b.log 2>&1; grep config gpurun_out/r27_n2b.log
$T --nproc-per-node 4 --master-port 29703 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r27_n4.log 2>&1; grep config gpurun_out/r27_n4.log
$T --nproc-per-node 4 --master-port 29704 tools/bench_configs.py --configs mnist60k,har200k --iters 10 --grid-rows 2 > gpurun_out/r27_n4g.log 2>&1; grep config gpurun_out/r27_n4g.log
$T --nproc-per-node 4 --master-port 29705 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r27_n4b.log 2>&1; grep config gpurun_out/r27_n4b.log
$T --nproc-per-node 4 --master-port 29706 tools/bench_configs.py --configs mnist1m --iters 3 --grid-rows 2 > gpurun_out/r27_n4c.log 2>&1; grep config gpurun_out/r27_n4c.log
$T --nproc-per-node 4 --master-port 29707 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r27_bench4.log 2>&1; tail -n 1 gpurun_out/r27_bench4.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29708 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r27_bench2.log 2>&1; tail -n 1 gpurun_out/r27_bench2.log | cut -c1-200
