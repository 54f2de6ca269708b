"""Per-iteration, per-rank phase times (a2 / a3 / a4, CUDA events inside kkm_fit) of one
config (a2 also split into the kernel and the rest): fit() is called with max_iter = 1 repeatedly and phase_ms() differenced. Launch with
torchrun for N > 1. Diagnoses one-time costs and rank imbalance (e.g. the 1.5D a3 time)."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mnist60k")
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--grid-rows", type=int, default=1)
ap.add_argument("--path", default="auto", choices=["auto", "mat", "stream"])
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
comm = None
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    uid = [kkm.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = kkm.comm_init(world, rank, uid[0])
cfg = dict(synth.CONFIGS[a.config])
n = cfg["n"]
r0, r1 = kkm.shard_begin(n, rank, world), kkm.shard_begin(n, rank + 1, world)
gen = synth.row_generator(a.config, n)
gamma = cfg.get("gamma") or synth.median_gamma(gen, n, cfg["seed"])
Xd = torch.from_numpy(gen(np.arange(r0, r1))).to(dev)
path = {"auto": kkm.PATH_AUTO, "mat": kkm.PATH_MATERIALIZE, "stream": kkm.PATH_STREAM}[a.path]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h = kkm.KernelKMeans(Xd, n, cfg["k"], cfg["kind"], gamma, cfg.get("coef0", 0.0), cfg.get("degree", 1),
                     max_iter=1, rank=rank, nranks=world, comm=comm, timing=True, path=path,
                     grid_rows=a.grid_rows)
e1.record()
torch.cuda.synchronize()
init_ms = e0.elapsed_time(e1)
rows, prev = [], h.phase_ms()
for t in range(a.iters):
    h.fit()
    cur = h.phase_ms()
    rows.append([cur[p] - prev[p] for p in ("spmm", "cnorm", "assign", "a2_kernel")])
    prev = cur
mine = torch.tensor([[init_ms] + [x for r in rows for x in r]], dtype=torch.float64, device=dev)
if world > 1:
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    allr = torch.cat(allr).cpu().numpy()
else:
    allr = mine.cpu().numpy()
if rank == 0:
    for r in range(world):
        v = allr[r]
        its = v[1:].reshape(a.iters, 4)
        print(json.dumps({"config": a.config, "grid": f"{a.grid_rows}x{world // a.grid_rows}", "rank": r,
                          "init_ms": round(float(v[0]), 2),
                          "a2_ms": [round(float(x), 3) for x in its[:, 0]],
                          "a3_ms": [round(float(x), 3) for x in its[:, 1]],
                          "a4_ms": [round(float(x), 3) for x in its[:, 2]],
                          # the a2 kernel alone; a2 - a2_kernel = sort / exchange / reduction around it
                          "a2_kernel_ms": [round(float(x), 3) for x in its[:, 3]]}))
h.destroy()
if comm:
    kkm.comm_destroy(comm)
if world > 1:
    dist.destroy_process_group()
