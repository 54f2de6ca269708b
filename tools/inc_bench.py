"""f3 time to solution: one clustering run of a BASELINE config with and without the
incremental S update (kkm_params.incremental): per-iteration changed counts, a2 phase time and
total fit time (CUDA events), same seeds."""
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
ap.add_argument("--path", default="auto", choices=["auto", "mat", "stream"])
a = ap.parse_args()
X, cfg = synth.make_config(a.config, n=a.n or None)
iters = a.iters or cfg["iters"]
path = {"auto": kkm.PATH_AUTO, "mat": kkm.PATH_MATERIALIZE, "stream": kkm.PATH_STREAM}[a.path]
Xd = torch.from_numpy(X).cuda()
out = {}
for inc in (False, True, False, True):  # second pair after warm-up
    h = kkm.KernelKMeans(Xd, X.shape[0], cfg["k"], cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"],
                         max_iter=iters, path=path, timing=True, incremental=inc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    it, J, ch = h.fit()
    e1.record()
    torch.cuda.synchronize()
    out["incremental" if inc else "full"] = dict(fit_ms=round(e0.elapsed_time(e1), 2), iters=it,
                                                 a2_ms=round(h.phase_ms()["spmm"], 2), final_J=float(J[-1]),
                                                 changed=[int(c) for c in ch])
    h.destroy()
f, i = out["full"], out["incremental"]
print(json.dumps({"what": "f3 incremental S", "config": a.config, "n": X.shape[0], "k": cfg["k"], "path": a.path,
                  "iterations": iters, "fit_ms_full": f["fit_ms"], "fit_ms_incremental": i["fit_ms"],
                  "a2_ms_full": f["a2_ms"], "a2_ms_incremental": i["a2_ms"],
                  "speedup": round(f["fit_ms"] / i["fit_ms"], 2),
                  "J_rel_diff": abs(f["final_J"] - i["final_J"]) / abs(f["final_J"]),
                  "same_changed_trace": f["changed"] == i["changed"], "changed": i["changed"]}))
