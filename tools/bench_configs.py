"""Seconds per iteration and total clustering time for the BASELINE.json configs at N GPUs
(launch with torchrun for N > 1). One JSON line per config on rank 0; device-timed with CUDA
events, max over ranks. Not the driver's bench line (bench.py is); this fills BASELINE.md.

  python tools/bench_configs.py --configs rings,har200k --iters 5
  torchrun --nproc-per-node 4 tools/bench_configs.py --configs mnist1m --iters 3 --grid-rows 2
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="rings,mnist60k,har200k")
ap.add_argument("--iters", type=int, default=0, help="override iterations (0 = config's)")
ap.add_argument("--points", "--n", dest="n", type=int, default=0, help="override n (labelled in the output)")
ap.add_argument("--grid-rows", type=int, default=1)
ap.add_argument("--path", default="auto", choices=["auto", "mat", "stream"])
ap.add_argument("--symmetric", default="auto", choices=["auto", "off", "on"])
ap.add_argument("--k", type=int, default=0, help="override the cluster count (labelled in the output)")
ap.add_argument("--kstore", default="auto", choices=["auto", "fp32", "fp16", "fp16x2"],
                help="materialised band storage (f4: fp16 = low-precision storage)")
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
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
path = {"auto": kkm.PATH_AUTO, "mat": kkm.PATH_MATERIALIZE, "stream": kkm.PATH_STREAM}[a.path]

# warm-up: load every kernel module once on a tiny problem (lazy loading is per kernel, not per size)
for wpath in (kkm.PATH_MATERIALIZE, kkm.PATH_STREAM):
    for wk in (2, 6, 10):
        wn = 2048
        r0, r1 = kkm.shard_begin(wn, rank, world), kkm.shard_begin(wn, rank + 1, world)
        Xw = torch.from_numpy(synth.blobs(wn, 784, wk, seed=1, rows=np.arange(r0, r1))).to(dev)
        hw = kkm.KernelKMeans(Xw, wn, wk, kkm.KERNEL_GAUSSIAN, 1e-3, 0.0, 1, max_iter=1, rank=rank,
                              nranks=world, comm=comm, path=wpath, grid_rows=a.grid_rows)
        hw.fit()
        hw.destroy()
torch.cuda.synchronize()

for name in a.configs.split(","):
    cfg = dict(synth.CONFIGS[name])
    if a.k:
        cfg["k"] = a.k
    n = a.n or cfg["n"]
    iters = a.iters or cfg["iters"]
    t0 = time.time()
    r0, r1 = kkm.shard_begin(n, rank, world), kkm.shard_begin(n, rank + 1, world)
    gen = synth.row_generator(name, n)
    Xl = gen(np.arange(r0, r1))
    gamma = cfg.get("gamma")
    if gamma is None:
        gamma = synth.median_gamma(gen, n, cfg["seed"])
    gen_s = time.time() - t0
    Xd = torch.from_numpy(Xl).to(dev)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    h = kkm.KernelKMeans(Xd, n, cfg["k"], cfg["kind"], gamma, cfg.get("coef0", 0.0),
                         cfg.get("degree", 1), max_iter=iters, rank=rank, nranks=world, comm=comm,
                         timing=True, path=path, grid_rows=a.grid_rows,
                         symmetric={"auto": kkm.SYM_AUTO, "off": kkm.SYM_OFF, "on": kkm.SYM_ON}[a.symmetric],
                         kstore={"auto": kkm.KSTORE_AUTO, "fp32": kkm.KSTORE_FP32, "fp16": kkm.KSTORE_FP16,
                                 "fp16x2": kkm.KSTORE_FP16X2}[a.kstore])
    e1.record()
    it, J, ch = h.fit()
    e2.record()
    torch.cuda.synchronize()
    init_ms, fit_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
    ph = h.phase_ms()
    kfull = 4.0 * (-(-n // world)) * (-(-n // 32) * 32)  # full K rows of a rank
    mat = h.params.path == kkm.PATH_MATERIALIZE or (
        h.params.path == kkm.PATH_AUTO
        and kkm.workspace_size(h.params, n, Xl.shape[1], rank, world) > 0.3 * kfull)
    sym = (mat and (cfg["k"] <= 16 or (cfg["k"] <= 32 and a.kstore != "fp32")) and a.grid_rows <= 1
           and h.params.symmetric != kkm.SYM_OFF
           and (h.params.symmetric == kkm.SYM_ON or n >= 8192))  # make_plan's rule
    vals = torch.tensor([init_ms, fit_ms, ph["spmm"], ph["cnorm"], ph["assign"], ph["init_gemm"], ph["a2_kernel"]],
                        dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    init_ms, fit_ms, spmm_ms, cn_ms, as_ms, gemm_ms, a2k_ms = vals.tolist()
    if rank == 0:
        d = Xl.shape[1]
        B = -(-n // world)
        loop_ms = (spmm_ms + cn_ms + as_ms) / it
        out = {"config": name, "n": n, "d": d, "k": cfg["k"], "n_gpus": world, "kstore": a.kstore,
               "grid": f"{a.grid_rows}x{world // a.grid_rows}", "iterations": it,
               "path": ((("materialised (f1 bands, " + {"fp16": "fp16 plane", "fp32": "fp32"}.get(
                            a.kstore, "hi + lo fp16 planes") + (", a2 on tensor cores)" if a.kstore != "fp32" else ")"))
                         if sym else "materialised")
                        if mat else
                        ("streaming (f1 upper triangle)" if cfg["k"] <= 16 and a.grid_rows <= 1
                         else "streaming")),
               "sec_per_iter": loop_ms / 1e3, "total_clustering_s": (init_ms + fit_ms) / 1e3,
               "init_s": init_ms / 1e3, "phases_ms_per_iter": {"a2": spmm_ms / it, "a2_kernel": a2k_ms / it,
                                                             "a3": cn_ms / it, "a4": as_ms / it},
               "final_J": float(J[-1]), "gen_s": round(gen_s, 1)}
        useful = 2.0 * B * n * d
        if mat:
            ldk = -(-n // 32) * 32
            kbytes = B * ldk * 4  # full K rows of the rank
            if sym:  # the rank's share of the upper-triangle bands, at the storage's bytes per value
                kbytes = (n * (n + 1024) / 2) / world * (2 if a.kstore == "fp16" else 4)
            gbs = kbytes / (spmm_ms / it * 1e-3) / 1e9
            out["a2_roofline"] = {"achieved_GBs": gbs, "frac_of_measured_hbm": gbs / peaks["hbm_gbs"]}
            if gemm_ms > 0:
                tf = useful / (gemm_ms * 1e-3) / 1e12
                out["a1_roofline"] = {"achieved_useful_TFs": tf,
                                      "frac_of_measured_bf16_div3": tf / (peaks["bf16_tflops"] / 3)}
        else:
            tf = useful / (spmm_ms / it * 1e-3) / 1e12
            out["a1a2_roofline"] = {"achieved_useful_TFs": tf,
                                    "frac_of_measured_bf16_div3": tf / (peaks["bf16_tflops"] / 3)}
        print(json.dumps(out), flush=True)
    h.destroy()
    del Xd
    torch.cuda.empty_cache()
if comm:
    kkm.comm_destroy(comm)
if world > 1:
    dist.destroy_process_group()
