# 4 GPUs, config 2: the peer-memory exchange vs the NCCL allreduce of S (KKM_NO_P2P=1), phase split per iteration
mkdir -p gpurun_out
make > /dev/null 2>&1 || { echo make failed; exit 1; }
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export KKM_NO_P2P=1; else unset KKM_NO_P2P; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2970$v bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r109_bench4_$v.log 2>&1; echo "bench4 nop2p=$v rc=$?"
  tail -1 gpurun_out/r109_bench4_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d.get('phases_ms_per_step'),d['clocks']['sm_mhz'])"
done
