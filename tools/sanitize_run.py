"""Small end-to-end runs of every hot kernel family for compute-sanitizer (one tool per gpurun call):
the chained band GEMM + spmm_tc (16 and 32 labels), fp32 bands (spmm_sym), full K (spmm_onehot / group),
the streaming f1 kernel (ssym), the full streaming kernel (tc3_stream), predict and the f3 deltas."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_17136_b200 as kkm  # noqa: E402
import synth  # noqa: E402

X, cfg = synth.make_config("mnist60k", n=3001)
Xd = torch.from_numpy(X).cuda()
runs = [dict(k=10, path=kkm.PATH_MATERIALIZE, symmetric=kkm.SYM_ON),                               # spmm_tc<16>
        dict(k=24, path=kkm.PATH_MATERIALIZE, symmetric=kkm.SYM_ON),                               # spmm_tc<32>
        dict(k=10, path=kkm.PATH_MATERIALIZE, symmetric=kkm.SYM_ON, kstore=kkm.KSTORE_FP32),       # spmm_sym
        dict(k=21, path=kkm.PATH_MATERIALIZE, symmetric=kkm.SYM_OFF),                              # group SpMM
        dict(k=10, path=kkm.PATH_STREAM),                                                          # ssym
        dict(k=10, path=kkm.PATH_STREAM, symmetric=kkm.SYM_OFF, incremental=True)]                 # tc3_stream
for kw in runs:
    k = kw.pop("k")
    h = kkm.KernelKMeans(Xd, 3001, k, kkm.KERNEL_GAUSSIAN, 0.02, 0.0, 1, max_iter=3, **kw)
    it, J, ch = h.fit()
    lab = h.predict(Xd[:257])
    print(k, kw, it, float(J[-1]), int(lab.sum()), flush=True)
    h.destroy()
torch.cuda.synchronize()
print("SANITIZE RUN OK")
