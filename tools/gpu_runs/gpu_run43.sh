mkdir -p gpurun_out
make -B > gpurun_out/r43_build.log 2>&1 || { tail -20 gpurun_out/r43_build.log; exit 1; }
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/r43_pytest.log 2>&1; tail -2 gpurun_out/r43_pytest.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29741 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r43_n2b.log 2>&1
$T --nproc-per-node 4 --master-port 29742 tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r43_n4b.log 2>&1
$T --nproc-per-node 4 --master-port 29743 tools/bench_configs.py --configs mnist1m --iters 3 --grid-rows 2 > gpurun_out/r43_n4g.log 2>&1
$T --nproc-per-node 4 --master-port 29744 tools/bench_configs.py --configs mnist8m --iters 1 > gpurun_out/r43_n4c.log 2>&1
grep -h '^{"config"' gpurun_out/r43_n*.log | cut -c1-220
