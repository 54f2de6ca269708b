"""Signed error of the a1 GEMM (linear kernel) vs fp64, per precision: mean relative bias and
max relative error of b = x.y, on the MNIST-like and HAR-like recipes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

for name, n in [("mnist60k", 1024), ("har200k", 1024)]:
    X, cfg = synth.make_config(name, n=n)
    Kr = oracle.kernel_matrix(X, oracle.LINEAR)
    for pname, prec in [("fp32", kkm.PREC_FP32_SIMT), ("fp16x3", kkm.PREC_FP16X3), ("bf16x3", kkm.PREC_BF16X3)]:
        h = kkm.KernelKMeans(torch.from_numpy(X).cuda(), n, 2, kkm.KERNEL_LINEAR, 1.0, 0.0, 1,
                             max_iter=1, precision=prec)
        Kg = h.kernel_tile(0, 0, n, n).astype(np.float64)
        scale = np.sqrt(np.outer(np.diag(Kr), np.diag(Kr)))
        rel = (Kg - Kr) / np.maximum(scale, 1e-30)
        print(f"{name:9s} {pname:7s} mean signed {rel.mean():+.3e}  mean|.| {np.abs(rel).mean():.3e}  max|.| {np.abs(rel).max():.3e}")
        h.destroy()
