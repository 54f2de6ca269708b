"""Objective precision at convergence: fit a BASELINE config with the tensor-core path, then
evaluate J of the final labels with the fp32 CUDA-core path (no systematic accumulation bias)
and report the relative difference (north_star: final objective within 1e-5)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mnist60k")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--precision", default="fp16x3")
ap.add_argument("--symmetric", default="auto")
a = ap.parse_args()
X, cfg = synth.make_config(a.config, n=a.n or None)
n = X.shape[0]
iters = a.iters or cfg["iters"]
args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
Xd = torch.from_numpy(X).cuda()
prec = {"fp16x3": kkm.PREC_FP16X3, "bf16x3": kkm.PREC_BF16X3}[a.precision]
sym = {"auto": kkm.SYM_AUTO, "off": kkm.SYM_OFF}[a.symmetric]
h = kkm.KernelKMeans(Xd, n, cfg["k"], *args, max_iter=iters, precision=prec, symmetric=sym)
it, J, ch = h.fit()
lab = h.assign()
J_tc = h.objective()
h.destroy()
torch.cuda.empty_cache()
hs = kkm.KernelKMeans(Xd, n, cfg["k"], *args, max_iter=1, precision=kkm.PREC_FP32_SIMT, symmetric=sym,
                      init_labels=lab.cpu().numpy())
J_ref = hs.objective()
diag = hs.debug_read(kkm.DBG_DIAG)
print(json.dumps({"config": a.config, "n": n, "iters": it, "precision": a.precision, "symmetric": a.symmetric,
                  "J_tc": J_tc, "J_fp32simt": J_ref, "rel_diff": (J_tc - J_ref) / abs(J_ref),
                  "J_over_trK": J_ref / float(diag.sum()), "changed_last": int(ch[-1]) if len(ch) else None}))
