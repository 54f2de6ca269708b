make > /dev/null 2>&1 || exit 1
timeout 900 python tools/bench_configs.py --configs rings,mnist60k,har200k > gpurun_out/r83_cfg1.jsonl 2> gpurun_out/r83_cfg1.err; cat gpurun_out/r83_cfg1.jsonl | cut -c1-250
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N tools/bench_configs.py --configs mnist60k,har200k > gpurun_out/r83_cfg$N.jsonl 2> gpurun_out/r83_cfg$N.err; cat gpurun_out/r83_cfg$N.jsonl | cut -c1-250
done
