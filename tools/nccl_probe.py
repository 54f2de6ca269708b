"""Per-call device time of the collectives the 1D f1 exchange could use, at config-2 sizes
(n = 60000, k = 10): allreduce of the int64 S (4.8 MB) vs fp64 / fp32, reduce-scatter of it,
the labels allgather and a (k + 1)-double allreduce. torchrun, one rank per GPU; prints rank 0's
median over reps (CUDA events on the current stream, after warm-up)."""
import json
import os
import statistics

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n, k, reps = 60000, 10, 50


def timeit(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


out = {"world": world}
for name, dt in (("int64", torch.int64), ("float64", torch.float64), ("float32", torch.float32)):
    x = torch.ones(n * k, dtype=dt, device="cuda")
    out[f"allreduce_{name}_us"] = timeit(lambda: dist.all_reduce(x))
xs = torch.ones(n * k, dtype=torch.int64, device="cuda")
ys = torch.empty(n * k // world, dtype=torch.int64, device="cuda")
out["reduce_scatter_int64_us"] = timeit(lambda: dist.reduce_scatter_tensor(ys, xs))
lab = torch.zeros(n, dtype=torch.int32, device="cuda")
out["allgather_labels_us"] = timeit(lambda: dist.all_gather_into_tensor(lab, lab[rank * (n // world):(rank + 1) * (n // world)]))
small = torch.ones(k + 1, dtype=torch.float64, device="cuda")
out["allreduce_k1_f64_us"] = timeit(lambda: dist.all_reduce(small))
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
