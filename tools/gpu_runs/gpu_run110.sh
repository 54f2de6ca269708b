# peer exchange only up to KKM_P2P_MAX_RANKS (default 4) ranks: the GPU tests on 4 GPUs, then run_multi
# on 4 GPUs with the default (peer) and with the threshold at 2 (the NCCL allreduce that P > 4 takes)
mkdir -p gpurun_out
make > /dev/null 2>&1 || { echo make failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r110_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r110_pytest.log
for m in 4 2; do
KKM_P2P_MAX_RANKS=$m timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$m tools/run_multi.py > gpurun_out/r110_multi4_$m.log 2>&1; echo "multi4 max=$m rc=$?"; grep -E "MULTI|36001" gpurun_out/r110_multi4_$m.log | cut -c1-200
done
