mkdir -p gpurun_out
make -B > gpurun_out/r55_build.log 2>&1 || { tail -20 gpurun_out/r55_build.log; exit 1; }
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r55_pytest.log 2>&1; tail -2 gpurun_out/r55_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r55_bench1.log 2>&1; tail -1 gpurun_out/r55_bench1.log | cut -c1-150
$T --nproc-per-node 2 --master-port 29761 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r55_bench2.log 2>&1; tail -1 gpurun_out/r55_bench2.log | cut -c1-150
$T --nproc-per-node 4 --master-port 29762 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r55_bench4.log 2>&1; tail -1 gpurun_out/r55_bench4.log | cut -c1-150
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r55_ref.log 2>&1; tail -1 gpurun_out/r55_ref.log | cut -c1-200
