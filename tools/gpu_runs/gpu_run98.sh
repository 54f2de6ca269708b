make > /dev/null 2>&1 || exit 1
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 tools/bench_configs.py --configs mnist8m --iters 2 > gpurun_out/r98_cfg5.jsonl 2> gpurun_out/r98_cfg5.err; grep -v NCCL gpurun_out/r98_cfg5.jsonl | cut -c1-600; tail -2 gpurun_out/r98_cfg5.err
