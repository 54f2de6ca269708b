mkdir -p gpurun_out
make -B > gpurun_out/r36_build.log 2>&1 || { tail -20 gpurun_out/r36_build.log; exit 1; }
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multi_gpu.py -q 2>&1 | tail -1
timeout 900 python tools/bench_configs.py --configs rings,mnist60k,har200k --iters 10 > gpurun_out/r36_n1.log 2>&1; grep config gpurun_out/r36_n1.log | cut -c1-300
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29721 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r36_n2.log 2>&1; grep config gpurun_out/r36_n2.log | cut -c1-300
$T --nproc-per-node 4 --master-port 29722 tools/bench_configs.py --configs mnist60k,har200k --iters 10 > gpurun_out/r36_n4.log 2>&1; grep config gpurun_out/r36_n4.log | cut -c1-300
$T --nproc-per-node 4 --master-port 29723 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r36_bench4.log 2>&1; tail -n 1 gpurun_out/r36_bench4.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29724 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r36_bench2.log 2>&1; tail -n 1 gpurun_out/r36_bench2.log | cut -c1-200
