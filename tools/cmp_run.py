"""Run a fixed reconstruction with the library in VDAMP_LIB and save x_hat (bitwise A/B of two builds).

    VDAMP_LIB=... python tools/cmp_run.py out.npz [config] [batch] [iters]
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1911_01234_b200 import vdamp, workload
out = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg1"
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 8
it = int(sys.argv[4]) if len(sys.argv) > 4 else 30
w = workload.make_workload(cfg, batch=nb)
res = {}
for prec in ("fp32", "fp64"):
    x, tr = vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, w.config.scales, it, ground_truths=w.x0, precision=prec)
    res[prec] = x
    res[prec + "_thr"] = np.array([[r.thresholds for r in t.records] for t in tr])
np.savez(out, **res)
