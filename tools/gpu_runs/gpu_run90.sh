make > /dev/null 2>&1 || exit 1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 tools/bench_configs.py --configs mnist1m --iters 5 > gpurun_out/r90_cfg4.jsonl 2> gpurun_out/r90_cfg4.err; cut -c1-400 gpurun_out/r90_cfg4.jsonl; tail -3 gpurun_out/r90_cfg4.err
