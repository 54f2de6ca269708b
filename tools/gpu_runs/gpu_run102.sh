make > /dev/null 2>&1 || exit 1
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2965$N tools/run_multi.py > gpurun_out/r102_multi$N.log 2>&1; echo "rc=$?"; grep -E "MULTI" gpurun_out/r102_multi$N.log
done
# p2p at a size where a3fix applies (n > 32768): 1D f1 bands, 2 GPUs vs 1 GPU
cat > /tmp/p2pcheck.py <<'PY'
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_2601_17136_b200 as kkm, synth
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
torch.cuda.set_device(rank); dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
uid = [kkm.get_unique_id() if rank == 0 else None]; dist.broadcast_object_list(uid, src=0)
comm = kkm.comm_init(world, rank, uid[0])
for name, n in (("har200k", 40000), ("mnist60k", 36001)):
    X, cfg = synth.make_config(name, n=n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    r0, r1 = kkm.shard_begin(n, rank, world), kkm.shard_begin(n, rank + 1, world)
    h = kkm.KernelKMeans(torch.from_numpy(X[r0:r1]).cuda(), n, cfg["k"], *args, max_iter=8, rank=rank, nranks=world, comm=comm)
    it, J, ch = h.fit(); lab = h.assign().cpu().numpy(); Jo = h.objective()
    if rank == 0:
        one = kkm.KernelKMeans(torch.from_numpy(X).cuda(), n, cfg["k"], *args, max_iter=8)
        it1, J1, _ = one.fit(); lab1 = one.assign().cpu().numpy()
        print(name, n, "P", world, "J identical", np.array_equal(J, J1), "labels identical", np.array_equal(lab, lab1), "objective", Jo == J[-1], flush=True)
    h.destroy(); dist.barrier()
kkm.comm_destroy(comm); dist.destroy_process_group()
PY
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2966$N /tmp/p2pcheck.py 2>&1 | grep -E "identical|Error|error" | head -5
done
