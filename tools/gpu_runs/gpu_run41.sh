mkdir -p gpurun_out
make -B > gpurun_out/r41_build.log 2>&1 || { tail -20 gpurun_out/r41_build.log; exit 1; }
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r41_pytest.log 2>&1; tail -2 gpurun_out/r41_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r41_bench1.log 2>&1; tail -1 gpurun_out/r41_bench1.log | cut -c1-150
timeout 900 python tools/bench_configs.py --configs rings,mnist60k,har200k --iters 10 > gpurun_out/r41_n1.log 2>&1
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r41_n1b.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29731 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r41_n2b.log 2>&1
$T --nproc-per-node 4 --master-port 29732 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r41_n4b.log 2>&1
$T --nproc-per-node 4 --master-port 29733 tools/bench_configs.py --configs mnist8m --iters 1 > gpurun_out/r41_n4c.log 2>&1
grep -h '^{"config"' gpurun_out/r41_n*.log | cut -c1-200
$T --nproc-per-node 4 --master-port 29734 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r41_bench4.log 2>&1; tail -n 1 gpurun_out/r41_bench4.log | cut -c1-150
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29735 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r41_bench2.log 2>&1; tail -n 1 gpurun_out/r41_bench2.log | cut -c1-150
