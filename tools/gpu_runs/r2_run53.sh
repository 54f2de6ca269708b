# round 2, 4 GPUs: one-box scaling curves of the final build -- bench.py (config 2) at N = 1, 2, 4 and
# config 4 (n = 1M, streaming f1) at N = 1, 2, 4, back to back
mkdir -p gpurun_out
make > gpurun_out/r2_53_make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python bench.py --no-cpu-baseline --stream-iters 0 > gpurun_out/r2_53_bench1.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/r2_53_bench1.log | cut -c1-120
for g in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2983$g bench.py --gpus $g --steps 5 --warmup 3 > gpurun_out/r2_53_bench$g.log 2>&1; echo "bench$g rc=$?"; tail -1 gpurun_out/r2_53_bench$g.log | cut -c1-120
done
timeout 900 python tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r2_53_c4_1.log 2>&1; echo "c4 x1 rc=$?"; grep '^{' gpurun_out/r2_53_c4_1.log | cut -c1-300
for g in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 --master-port 2984$g tools/bench_configs.py --configs mnist1m --iters 3 > gpurun_out/r2_53_c4_$g.log 2>&1; echo "c4 x$g rc=$?"; grep '^{' gpurun_out/r2_53_c4_$g.log | cut -c1-300
done
