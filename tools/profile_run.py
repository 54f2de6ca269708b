"""One clustering run of a BASELINE config for profiling (ncu) and error studies."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mnist60k")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--precision", default="fp16x3")
ap.add_argument("--path", default="auto", choices=["auto", "mat", "stream"])
ap.add_argument("--k", type=int, default=0, help="override the cluster count")
ap.add_argument("--full-k", action="store_true", help="store full K rows (KKM_SYM_OFF) instead of the f1 bands")
ap.add_argument("--kstore", default="auto", choices=["auto", "fp32", "fp16", "fp16x2"],
                help="materialised band storage (auto: hi + lo fp16 planes with a tensor-core precision)")
a = ap.parse_args()
X, cfg = synth.make_config(a.config, n=a.n or None)
prec = {"fp16x3": kkm.PREC_FP16X3, "bf16x3": kkm.PREC_BF16X3, "fp32": kkm.PREC_FP32_SIMT}[a.precision]
path = {"auto": kkm.PATH_AUTO, "mat": kkm.PATH_MATERIALIZE, "stream": kkm.PATH_STREAM}[a.path]
if a.k:
    cfg["k"] = a.k
h = kkm.KernelKMeans(torch.from_numpy(X).cuda(), X.shape[0], cfg["k"], cfg["kind"], cfg["gamma"],
                     cfg["coef0"], cfg["degree"], max_iter=a.iters, precision=prec, timing=True, path=path,
                     symmetric=kkm.SYM_OFF if a.full_k else kkm.SYM_AUTO,
                     kstore={"auto": kkm.KSTORE_AUTO, "fp32": kkm.KSTORE_FP32, "fp16": kkm.KSTORE_FP16,
                             "fp16x2": kkm.KSTORE_FP16X2}[a.kstore])
it, J, ch = h.fit()
torch.cuda.synchronize()
ph = h.phase_ms()
n, d = X.shape
flops = 2.0 * n * n * d
print(f"{a.config} n={n} d={d} path={a.path} iters {it} J {J[-1]:.6e} phases {ph}")
if a.path == "stream":
    per = ph["spmm"] / it
    line = f"stream a1+a2 per iteration {per:.2f} ms -> effective {flops / (per * 1e-3) / 1e12:.1f} TFLOP/s (2 n^2 d)"
    if not a.full_k and cfg["k"] <= 16:  # f1: only the upper-triangle pair tiles are computed
        T = -(-n // 256)
        ex = 2.0 * d * 256 * 256 * T * (T + 1) / 2
        line += f", executed {ex / (per * 1e-3) / 1e12:.1f} TFLOP/s (upper-triangle tiles)"
    print(line)
else:
    sym = not a.full_k and cfg["k"] <= 16
    eb = 2 if a.kstore == "fp16" else 4
    if sym:  # f1 bands: ~n^2/2 useful flops and K bytes
        TB, kb = 1024, 0
        for I in range(-(-n // TB)):
            kb += min(TB, n - I * TB) * (-(-(n - I * TB) // 32) * 32) * eb
        flops = 2.0 * d * kb / eb
    else:
        kb = n * (-(-n // 32) * 32) * 4
    print(f"a1 GEMM {ph['init_gemm']:.2f} ms -> useful {flops / (ph['init_gemm'] * 1e-3) / 1e12:.1f} TFLOP/s"
          f" ({'f1 bands' if sym else 'full K'})")
    per = ph["spmm"] / it
    print(f"a2 SpMM k={cfg['k']} {per:.3f} ms/iter -> K bytes {kb / 1e9:.2f} GB: {kb / (per * 1e-3) / 1e9:.0f} GB/s"
          f" (a2 kernel {ph['a2_kernel'] / it:.3f} ms: {kb / (ph['a2_kernel'] / it * 1e-3) / 1e9:.0f} GB/s)")
