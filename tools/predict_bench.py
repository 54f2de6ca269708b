"""Timing of kkm_predict: train on a BASELINE config's recipe, then assign m
held-out rows of the same recipe. Device-resident Y, CUDA events around the call (which
includes Y's split/prep, the label sort of X, the fused streaming kernel and the argmin), after
warm-up. Useful flops = 2 m n d; peak = measured dense bf16 / 3 (3 MMAs per product)."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mnist60k")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--m", type=int, default=60000)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--path", default="auto", choices=["auto", "mat", "stream"])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
Xa, cfg = synth.make_config(a.config, n=(a.n or synth.CONFIGS[a.config]["n"]) + a.m)
n = Xa.shape[0] - a.m
X, Y = torch.from_numpy(Xa[:n]).cuda(), torch.from_numpy(Xa[n:]).cuda()
k = a.k or cfg["k"]
path = {"auto": kkm.PATH_AUTO, "mat": kkm.PATH_MATERIALIZE, "stream": kkm.PATH_STREAM}[a.path]
h = kkm.KernelKMeans(X, n, k, cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"], max_iter=3, path=path)
h.fit()
for _ in range(2):
    lab = h.predict(Y)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
for _ in range(a.reps):
    lab = h.predict(Y)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
d = X.shape[1]
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
bf16 = peaks["bf16_tflops"]
tf = 2.0 * a.m * n * d / (ms * 1e-3) / 1e12
print(json.dumps({"what": "kkm_predict", "config": a.config, "n_train": n, "m": a.m, "d": d, "k": k,
                  "path": a.path, "ms": round(ms, 3), "points_per_s": round(a.m / (ms * 1e-3)),
                  "useful_tflops": round(tf, 1), "peak_useful_tflops": round(bf16 / 3, 1),
                  "frac": round(tf / (bf16 / 3), 3),
                  "labels_hist": torch.bincount(lab.long(), minlength=k).tolist()}))
h.destroy()
