python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r103_build.log 2>&1 || { tail -5 gpurun_out/r103_build.log; exit 1; }
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r103_pytest.log 2>&1; tail -1 gpurun_out/r103_pytest.log
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r103_bench$N.log 2>&1; tail -1 gpurun_out/r103_bench$N.log | cut -c1-120
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r103_bench1.log 2>&1; tail -1 gpurun_out/r103_bench1.log | cut -c1-120
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r103_ref.log 2>&1; tail -1 gpurun_out/r103_ref.log | cut -c1-160
