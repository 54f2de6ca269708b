#!/usr/bin/env python
"""Benchmark of the Kernel K-means hot path (BASELINE.json metric: sec/iteration and total
clustering time, % of roofline).

  python bench.py --gpus N --steps K --warmup W [--impl ours|reference]

A step is one whole clustering run of the hot path (all SURVEY §8(a) rows): kkm_init
(X resident on the device -> norms, bf16 split, diag, K = kappa(X X^T) materialised) and
kkm_fit (max_iter iterations of a2 SpMM, a3 cnorm/J, a4 distances/argmin/sizes, with the
1D exchange steps when N > 1) -> labels resident on the device. Workload: BASELINE.json
configs[1] (MNIST-shaped n=60000, d=784, k=10, poly(1,1,2), K materialised, 100 iterations
per P:639), synthetic and seeded (synth/). N > 1 shards the same n over N GPUs (strong
scaling). Inputs are far larger than L2 (K = 14.4 GB is streamed every iteration).

--impl reference runs the fp64 CPU oracle (oracle/) as it stands on the host cores on a
bounded row sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOAD = "mnist60k"
METRIC = "sec/iteration"


def workload_desc(cfg, iters):
    return (f"{WORKLOAD}: MNIST-shaped synthetic n={cfg['n']} d=784 k={cfg['k']} "
            f"poly(gamma=1,c=1,deg=2), K materialised (upper-triangle bands unless --symmetric off), "
            f"{iters} iterations (BASELINE.json configs[1])")


def bench_config(cfg, iters):
    """The workload both arms report (identical dicts, so the driver can pair the lines)."""
    return {"workload": workload_desc(cfg, iters), "n": cfg["n"], "d": 784, "k": cfg["k"],
            "iterations": iters, "l2": "inputs larger than L2 (the stored K is streamed every iteration)"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def sym_band_share(n, world, rank, TB=1024):
    """f1 band storage (csrc/sym.cuh, make_plan): bands of TB rows x ceil32(n - I TB) columns,
    largest first to the least-loaded rank. Returns (stored floats, useful flops / d / 2) of
    `rank` = its K bytes / 4 and GEMM products."""
    load = [0.0] * world
    mine = 0
    for I in range(-(-n // TB)):
        rows = min(TB, n - I * TB)
        ldb = -(-(n - I * TB) // 32) * 32
        r = min(range(world), key=lambda q: (load[q], q))
        load[r] += rows * ldb
        if r == rank:
            mine += rows * ldb
    return mine


def peaks_bf16_burst():
    p, _ = measured_peaks()
    return p["bf16_tflops"]


def cores():
    return len(os.sched_getaffinity(0))


# ------------------------------------------------------------------ CPU oracle (baseline)
def oracle_sample(X, cfg, rows_n=1024, seed=0):
    """Bounded sample of the same workload on the fp64 oracle: exact K rows for `rows_n`
    random rows (a1) and one E / c / D / argmin pass over them (a2-a4), extrapolated to n."""
    import oracle
    n, k = X.shape[0], cfg["k"]
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    rows = np.sort(np.random.default_rng(seed).choice(n, rows_n, replace=False))
    labels = oracle.round_robin(n, k)
    t0 = time.perf_counter()
    Kr = oracle.kernel_rows(X, rows, *args)
    t1 = time.perf_counter()
    E = oracle.E_rows(Kr, labels, k)
    diag = oracle.kernel_diag(X, *args, rows=rows)
    cn = np.array([E[labels[rows] == c, c].mean() if (labels[rows] == c).any() else 0.0
                   for c in range(k)])
    oracle.assign(E, diag, cn)
    t2 = time.perf_counter()
    per_iter = (t2 - t1) * n / rows_n
    k_build = (t1 - t0) * n / rows_n
    return dict(sec_per_iter=per_iter, k_build_s=k_build, wall_s=t2 - t0, rows=rows_n)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    X, cfg = synth.make_config(WORKLOAD)
    iters = args.iters or cfg["iters"]
    # rank 0 runs alone (the other ranks exit above), so it takes every host core: torchrun's
    # OMP_NUM_THREADS=1 default (set against oversubscription) is replaced before the oracle's
    # OpenMP runtime loads; an explicit setting on a 1-process run is kept
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or "OMP_NUM_THREADS" not in os.environ:
        os.environ["OMP_NUM_THREADS"] = str(cores())
    threads = int(os.environ["OMP_NUM_THREADS"])
    for _ in range(args.warmup):
        oracle_sample(X, cfg, args.ref_rows)
    samples = [oracle_sample(X, cfg, args.ref_rows, seed=s) for s in range(args.steps)]
    spi = statistics.mean(s["sec_per_iter"] for s in samples)
    kb = statistics.mean(s["k_build_s"] for s in samples)
    total = kb + iters * spi
    sample = (f"{args.ref_rows} of {cfg['n']} rows per step: exact fp64 K rows + one E/c/D/argmin "
              f"pass, extrapolated x n/{args.ref_rows} (OMP threads={threads})")
    line = {
        "impl": "reference", "metric": METRIC, "value": spi, "unit": "s/iteration",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(s["wall_s"] for s in samples),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "total_clustering_s": total,
        "config": bench_config(cfg, iters),
        "parallelism": "cpu-oracle",
        "cpu_baseline": {"value": spi, "unit": "s/iteration", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": spi, "unit": "s/iteration", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({nm for r in self.rows for nm, v in zip(names, r[4:8]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2601_17136_b200 as kkm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = None
    if world > 1:
        uid = [kkm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = kkm.comm_init(world, rank, uid[0])

    cfg = dict(synth.CONFIGS[WORKLOAD])
    n, k = cfg["n"], cfg["k"]
    iters = args.iters or cfg["iters"]
    r0, r1 = kkm.shard_begin(n, rank, world), kkm.shard_begin(n, rank + 1, world)
    X_local = synth.mnist_like(n, cfg["seed"], row_begin=r0, row_end=r1)
    d = X_local.shape[1]
    precision = {"bf16x3": kkm.PREC_BF16X3, "fp16x3": kkm.PREC_FP16X3,
                 "fp32": kkm.PREC_FP32_SIMT}[args.precision]
    kw = dict(kind=cfg["kind"], gamma=1.0, coef0=1.0, degree=2, max_iter=iters,
              precision=precision, rank=rank, nranks=world, comm=comm, timing=True,
              symmetric=kkm.SYM_AUTO if args.symmetric == "auto" else kkm.SYM_OFF,
              kstore={"auto": kkm.KSTORE_AUTO, "fp32": kkm.KSTORE_FP32, "fp16x2": kkm.KSTORE_FP16X2}[args.kstore])
    p = kkm.default_params()
    p.kind, p.k, p.max_iter, p.precision = cfg["kind"], k, iters, precision
    p.symmetric = kw["symmetric"]
    p.kstore = kw["kstore"]
    ws = torch.empty(kkm.workspace_size(p, n, d, rank, world), dtype=torch.uint8, device=dev)
    Xd = torch.from_numpy(X_local).to(dev)
    Xh = torch.from_numpy(X_local).pin_memory()
    lab_h = torch.empty(n, dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def one_step(X_src, lab_dst=None):
        h = kkm.KernelKMeans(X_src, n, k, workspace=ws, stream=stream, **kw)
        it, J, ch = h.fit()
        if lab_dst is not None:
            h.assign(lab_dst)
        ph, nl = h.phase_ms(), h.launch_count()
        h.destroy()
        return it, J, ph, nl

    for _ in range(args.warmup):
        one_step(Xd)
    barrier()

    # ---- timed region: K steps, X resident in HBM
    phases, launches, J_last = [], 0, None
    with ClockSampler(local) as clk:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            it, J, ph, nl = one_step(Xd)
            phases.append(ph)
            launches += nl
            J_last = J
        ev1.record(stream)
        barrier()
    step_ms = ev0.elapsed_time(ev1) / args.steps
    clocks = clk.summary()

    # ---- e2e: the same through the C-ABI with HOST buffers (H2D of X, D2H of labels inside)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_step(Xh, lab_h)
    e1.record(stream)
    barrier()
    e2e_step_ms = e0.elapsed_time(e1) / args.steps

    # ---- informational, not the metric: the same clustering run with the f3 incremental S
    # update (kkm_params.incremental = 1; identical label trace), X resident,
    # its own (preallocated) workspace, after one untimed warm-up run
    p.incremental = 1
    ws_inc = torch.empty(kkm.workspace_size(p, n, d, rank, world), dtype=torch.uint8, device=dev)
    p.incremental = 0

    def inc_run():
        hinc = kkm.KernelKMeans(Xd, n, k, workspace=ws_inc, stream=stream, incremental=True, **kw)
        _, Jr, _ = hinc.fit()
        hinc.destroy()
        return Jr

    inc_run()
    barrier()
    i0 = torch.cuda.Event(enable_timing=True)
    i1 = torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    J_inc = inc_run()
    i1.record(stream)
    barrier()
    inc_ms = i0.elapsed_time(i1)
    del ws_inc

    # ---- informational, not the metric: the same run with f4 fp16 K storage (the bands in fp16,
    # a2 on the tensor cores; each K value rounded to 2^-11 relative, A27 -- below the
    # paper's fp32 precision, so never the headline)
    kh_ok = precision != kkm.PREC_FP32_SIMT and kw["symmetric"] == kkm.SYM_AUTO and k <= 32
    kh_ms = kh_a2 = kh_a2k = None
    J_kh = None
    if kh_ok:
        p.kstore = kkm.KSTORE_FP16
        ws_kh = torch.empty(kkm.workspace_size(p, n, d, rank, world), dtype=torch.uint8, device=dev)
        p.kstore = kw["kstore"]
        kw_kh = dict(kw, kstore=kkm.KSTORE_FP16)

        def kh_run():
            hk = kkm.KernelKMeans(Xd, n, k, workspace=ws_kh, stream=stream, **kw_kh)
            _, Jr, _ = hk.fit()
            phr = hk.phase_ms()
            hk.destroy()
            return Jr, phr

        kh_run()
        barrier()
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        J_kh, ph_kh = kh_run()
        k1.record(stream)
        barrier()
        kh_ms = k0.elapsed_time(k1)
        kh_a2, kh_a2k = ph_kh["spmm"] / iters, ph_kh["a2_kernel"] / iters
        del ws_kh

    # ---- informational, not the metric: the same run with the f1 bands stored in fp32 (the paper's
    # storage precision) and the one-hot FFMA2 a2 (sym.cuh), X resident, own workspace
    f32_ok = kw["kstore"] == kkm.KSTORE_AUTO and precision != kkm.PREC_FP32_SIMT and \
        kw["symmetric"] == kkm.SYM_AUTO and k <= 16
    f32_iter = f32_a2 = None
    J_f32 = None
    if f32_ok:
        p.kstore = kkm.KSTORE_FP32
        ws_f32 = torch.empty(kkm.workspace_size(p, n, d, rank, world), dtype=torch.uint8, device=dev)
        p.kstore = kw["kstore"]
        kw_f32 = dict(kw, kstore=kkm.KSTORE_FP32)

        def f32_run():
            hf = kkm.KernelKMeans(Xd, n, k, workspace=ws_f32, stream=stream, **kw_f32)
            _, Jr, _ = hf.fit()
            phr = hf.phase_ms()
            hf.destroy()
            return Jr, phr

        f32_run()
        barrier()
        J_f32, ph_f32 = f32_run()
        barrier()
        f32_iter = (ph_f32["spmm"] + ph_f32["cnorm"] + ph_f32["assign"]) / iters
        f32_a2 = ph_f32["spmm"] / iters
        del ws_f32

    # ---- informational, not the metric: the streaming path at the BASELINE configs[3] recipe
    # (n = 1,000,000, d = 784, k = 10, Gaussian, median gamma): K (4 TB) is never stored; every
    # iteration recomputes the upper triangle of the label-sorted K on the tensor cores (ssym.cuh).
    # One GPU only (rank 0 of a 1-GPU run), 1 untimed + `--stream-iters` timed iterations.
    stream_info = None
    if world == 1 and args.stream_iters > 0:
        scfg = synth.CONFIGS["mnist1m"]
        sn = scfg["n"]
        Xs = synth.mnist_like(sn, scfg["seed"])
        sgamma = synth.median_gamma(synth.row_generator("mnist1m"), sn, scfg["seed"])
        Xsd = torch.from_numpy(Xs).to(dev)
        del Xs
        ps = kkm.default_params()
        si = args.stream_iters
        ps.kind, ps.k, ps.max_iter, ps.precision, ps.timing = kkm.KERNEL_GAUSSIAN, scfg["k"], si, precision, 1
        ws_s = torch.empty(kkm.workspace_size(ps, sn, 784, 0, 1), dtype=torch.uint8, device=dev)
        hs = kkm.KernelKMeans(Xsd, sn, scfg["k"], kkm.KERNEL_GAUSSIAN, sgamma, 0.0, 1, max_iter=si, precision=precision,
                              workspace=ws_s, stream=stream, timing=True)
        hs.fit()  # warm-up fit (the same iterations: sort, kernel modules, clocks)
        ph0 = hs.phase_ms()
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as sclk:
            s0.record(stream)
            hs.fit()
            s1.record(stream)
            barrier()
        ph1 = hs.phase_ms()
        # sec/iteration of the loop (phase timers: a2 + a3 + a4 of the timed iterations; the fit's extra
        # objective pass for the final labels is outside, as in the metric's line)
        s_ms = sum(ph1[key] - ph0[key] for key in ("spmm", "cnorm", "assign")) / args.stream_iters
        fit_ms = s0.elapsed_time(s1)
        a2k = (ph1["a2_kernel"] - ph0["a2_kernel"]) / args.stream_iters
        T = -(-sn // 256)
        exec_flops = 2.0 * 784 * 256 * 256 * T * (T + 1) / 2  # the upper-triangle tiles the kernel computes
        paper_flops = 2.0 * sn * sn * 784                       # the paper's full K GEMM per iteration
        stream_info = {"workload": "mnist1m: BASELINE.json configs[3] recipe, n=1000000 d=784 k=10 Gaussian "
                                   "(median gamma), K streamed (never stored), 1 GPU",
                       "value": s_ms / 1e3, "unit": "s/iteration", "iterations_timed": args.stream_iters,
                       "fit_s": fit_ms / 1e3,
                       "kernel": "ssym_kernel (upper triangle of the label-sorted K, chained fp16x3 tcgen05)",
                       "kernel_ms": a2k,
                       "roofline": {"bound": "tensor", "unit": "TFLOP/s",
                                    "achieved": exec_flops / (a2k * 1e-3) / 1e12,
                                    "peak": peaks_bf16_burst() / 3.0,
                                    "frac": exec_flops / (a2k * 1e-3) / 1e12 / (peaks_bf16_burst() / 3.0),
                                    "traffic": None,
                                    "achieved_paper_equivalent": paper_flops / (a2k * 1e-3) / 1e12,
                                    "flops_per_launch_useful": exec_flops,
                                    # what the tensor pipe issues: 3 fp16 MMAs over the 64-padded depth
                                    "mma_issue_tflops": 3 * exec_flops * (-(-784 // 64) * 64) / 784 / (a2k * 1e-3) / 1e12,
                                    "mma_issue_frac_of_bf16_peak": 3 * exec_flops * (-(-784 // 64) * 64) / 784
                                    / (a2k * 1e-3) / 1e12 / peaks_bf16_burst(),
                                    "note": "useful = the upper-triangle tiles' 2 d flops per entry; fp16x3 = 3 dense "
                                            "16-bit MMAs per useful product, so peak = the measured bf16 dense (burst) "
                                            "figure / 3. The kernel runs seconds at the power cap and still exceeds "
                                            "the measured sustained figure / 3, so the burst one is the ceiling"},
                       "clocks": sclk.summary()}
        hs.destroy()
        del ws_s, Xsd
        torch.cuda.empty_cache()

    ph_mean = {key: statistics.mean(p_[key] for p_ in phases) for key in phases[0]}
    loop_ms = ph_mean["spmm"] + ph_mean["cnorm"] + ph_mean["assign"]
    vals = torch.tensor([inc_ms, step_ms, e2e_step_ms, loop_ms / iters, ph_mean["spmm"] / iters,
                         ph_mean["init_gemm"], ph_mean["a2_kernel"] / iters, kh_ms or 0.0, kh_a2 or 0.0,
                         kh_a2k or 0.0, f32_iter or 0.0, f32_a2 or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    (inc_ms, step_ms, e2e_step_ms, iter_ms, spmm_ms, gemm_ms, a2k_ms, kh_ms, kh_a2, kh_a2k, f32_iter,
     f32_a2) = vals.tolist()

    if rank == 0:
        peaks, peak_kind = measured_peaks()
        B = -(-n // world)
        nloc = min(B, n - 0)
        ldk = -(-n // 32) * 32
        sym = args.symmetric == "auto" and (k <= 16 or (k <= 32 and args.kstore != "fp32"))
        # the f1 bands as hi + lo fp16 planes with a2 on the tensor cores (KSTORE_AUTO's choice
        # for a tensor-core precision), or fp32 bands with the one-hot FFMA2 kernel
        tc_a2 = sym and args.kstore != "fp32" and precision != kkm.PREC_FP32_SIMT
        a2_kernel = ("spmm_tc_kernel (a2 on the tensor cores over the f1 bands as hi + lo fp16 planes)" if tc_a2
                     else "spmm_sym_kernel (a2 on the f1 fp32 bands)" if sym else "spmm_onehot_kernel (a2)")
        if sym:  # f1: the rank's upper-triangle bands (K read once; the column partials are
            # implementation traffic, visible in `traffic`) + S partials of all rows
            kfl = sym_band_share(n, world, 0)
            spmm_bytes = kfl * 4 + n * k * 8
            gemm_flops = 2.0 * kfl * d
        else:
            spmm_bytes = nloc * ldk * 4 + ldk * 4 + nloc * k * 8  # K block + labels + S partials
            gemm_flops = 2.0 * nloc * n * d
        kh_bytes = sym_band_share(n, world, 0) * 2 + n * k * 8 if kh_ok else None  # fp16 bands + S
        spmm_gbs = spmm_bytes / (spmm_ms * 1e-3) / 1e9          # the whole a2 phase
        a2k_gbs = spmm_bytes / (a2k_ms * 1e-3) / 1e9            # the dominant kernel alone
        gemm_tfs = gemm_flops / (gemm_ms * 1e-3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "spmm_traffic.json")
        if os.path.exists(tp):  # only an ncu capture of this same launch shape (per-launch bytes)
            with open(tp) as f:
                caps = json.load(f).get("captures", [])
            for cap in caps:
                if a2_kernel.startswith(cap.get("kernel", "").split("<")[0]) and \
                        abs(cap.get("algorithmic_bytes", 0) - spmm_bytes) <= 0.01 * spmm_bytes:
                    traffic = cap.get("bytes_per_launch")
        tensor = precision in (kkm.PREC_BF16X3, kkm.PREC_FP16X3)
        # 3 dense 16-bit MMAs per useful product: useful-flop peak = measured bf16 dense / 3
        # (fp16 and bf16 share the dense rate); SIMT: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz
        gemm_peak = peaks["bf16_tflops"] / 3.0 if tensor else 148 * 128 * 2 * 1.965e9 / 1e12
        line = {
            "metric": METRIC, "value": iter_ms / 1e3, "unit": "s/iteration",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": ("fp16x3-mma/f32-acc; K as hi+lo fp16 planes" if tc_a2 else
                      "fp16x3-mma/f32-acc; K fp32" if tensor else "f32"),
            "data": "synthetic",
            "total_clustering_s": step_ms / 1e3,
            "config": bench_config(cfg, iters),
            "impl_config": {"precision_a1": args.precision,
                            "k_storage": ("f1 bands as hi + lo fp16 planes (hi = RN(K 2^e), lo = RN(K 2^e - hi)): "
                                          "per-value relative error <= 2^-21 + 2^-24 (tests/test_kstore_bound.py; "
                                          "~3 bits coarser than fp32 storage, lo plane subnormal for tiny K), "
                                          "E/c/J accumulated in int64 fixed point / fp64; DESIGN A27" if tc_a2 else
                                          "fp32 f1 bands" if sym else "fp32 full K rows"),
                            "parallelism": f"1D row shards x{world}" if world > 1 else "single GPU"},
            "roofline": {"kernel": a2_kernel,
                         "bound": "hbm", "achieved": a2k_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": a2k_gbs / peaks["hbm_gbs"], "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_launch": spmm_bytes, "launch_ms": a2k_ms,
                         "timing": "CUDA events around the kernel's launches on the handle's stream, "
                                   "inside the timed steps (kkm_phase_ms a2_kernel)"},
            "roofline_a2_phase": {"what": ("S memset + spmm_tc + fixed-point S to fp64" if tc_a2 else
                                           "band_sort + spmm_sym + sym_colsum + sym_reduce" if sym
                                           else "a2 launches"), "achieved": spmm_gbs,
                                  "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": spmm_gbs / peaks["hbm_gbs"],
                                  "phase_ms": spmm_ms},
            "roofline_a1": {"kernel": f"gemm ({args.precision}) + kappa", "bound": "tensor"
                            if tensor else "alu",
                            "achieved": gemm_tfs, "peak": gemm_peak, "unit": "TFLOP/s",
                            "frac": gemm_tfs / gemm_peak, "flops_per_launch": gemm_flops,
                            "launch_ms": gemm_ms},
            "phases_ms_per_step": ph_mean,
            "f3_incremental_informational": {
                "total_clustering_s": inc_ms / 1e3, "s_per_iteration_amortised": inc_ms / 1e3 / iters,
                "final_J_rel_diff": abs(float(J_inc[-1]) - float(J_last[-1])) / abs(float(J_last[-1])),
                "note": "not the metric: the same run with the opt-in incremental S update (f3); "
                        "the metric keeps the paper's full recompute of E every iteration"},
            "f4_fp16_kstore_informational": None if not kh_ok else {
                "total_clustering_s": kh_ms / 1e3,
                "a2_phase_ms": kh_a2, "a2_kernel_ms": kh_a2k,
                "a2_kernel": "spmm_tc_kernel (tcgen05, fp16 bands)",
                "a2_kernel_bytes_per_launch": kh_bytes,
                "a2_kernel_achieved_gbs": kh_bytes / (kh_a2k * 1e-3) / 1e9,
                "a2_kernel_frac": kh_bytes / (kh_a2k * 1e-3) / 1e9 / peaks["hbm_gbs"],
                "final_J_rel_diff": abs(float(J_kh[-1]) - float(J_last[-1])) / abs(float(J_last[-1])),
                "note": "not the metric: f4 low-precision K storage (fp16 bands, a2 on the tensor cores); "
                        "K values carry 2^-11 relative rounding (DESIGN A27), below the paper's fp32"},
            "fp32_bands_informational": None if not f32_ok else {
                "value": f32_iter / 1e3, "unit": "s/iteration", "a2_phase_ms": f32_a2,
                "final_J_rel_diff": abs(float(J_f32[-1]) - float(J_last[-1])) / abs(float(J_last[-1])),
                "note": "not the metric: the same run with the f1 bands stored in fp32 (kstore FP32) and the "
                        "one-hot FFMA2 a2 (sym.cuh); the metric's hi + lo fp16 planes are fp32-class (~2^-22, "
                        "DESIGN A27) and pass the same parity rules"},
            "e2e": {"value": e2e_step_ms / 1e3 / iters, "unit": "s/iteration",
                    "note": "amortised over the step's iterations: H2D of X (pinned host) + K build + "
                            "the iteration loop + D2H of the labels, through the C-ABI",
                    "total_clustering_s": e2e_step_ms / 1e3,
                    "h2d_bytes_per_step": int(X_local.nbytes), "d2h_bytes_per_step": int(n * 4)},
            "stream_config4_informational": stream_info,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "final_J": float(J_last[-1]),
        }
        if world == 1 and not args.no_cpu_baseline:
            os.environ.setdefault("OMP_NUM_THREADS", str(cores()))  # (before the oracle's OpenMP loads)
            threads = int(os.environ["OMP_NUM_THREADS"])
            X, full_cfg = synth.make_config(WORKLOAD)
            s = oracle_sample(X, full_cfg, args.ref_rows)
            line["cpu_baseline"] = {
                "value": s["sec_per_iter"], "unit": "s/iteration", "cores": threads, "kind": "oracle",
                "sample": (f"{args.ref_rows} of {n} rows: exact fp64 K rows + one E/c/D/argmin pass, "
                           f"extrapolated x n/{args.ref_rows}; K build extrapolated {s['k_build_s']:.1f} s"),
                "total_clustering_s": s["k_build_s"] + iters * s["sec_per_iter"]}
        print(json.dumps(line), flush=True)

    if comm:
        kkm.comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--iters", type=int, default=0, help="override iterations per step")
    ap.add_argument("--precision", choices=["fp16x3", "bf16x3", "fp32"], default="fp16x3")
    ap.add_argument("--ref-rows", type=int, default=1024)
    ap.add_argument("--symmetric", choices=["auto", "off"], default="auto",
                    help="auto: upper-triangle K bands (f1); off: full K rows")
    ap.add_argument("--kstore", choices=["auto", "fp32", "fp16x2"], default="auto",
                    help="f1 band storage: auto = hi + lo fp16 planes (fp32-class, a2 on the tensor cores) "
                         "with a tensor-core precision; fp32 = fp32 bands (one-hot FFMA2 a2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stream-iters", type=int, default=2,
                    help="timed iterations of the informational 1M streaming line (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
    sys.exit(run_reference(args) if args.impl == "reference" else run_ours(args))


if __name__ == "__main__":
    main()
