import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_01234_b200 import vdamp, workload
w = workload.make_workload("cfg2", batch=32)
for prec in ("fp32",):
    t0 = time.time()
    xs, trs = vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 5, 50, ground_truths=w.x0, precision=prec)
    print(prec, "time", time.time() - t0, "finite", np.isfinite(xs).all())
    for b in range(32):
        tr = trs[b]
        al = np.array([r.alphas for r in tr.records]); cl = [r.alpha_clamped for r in tr.records]
        nm = tr.nmse_curve()
        if not np.isfinite(nm).all() or any(cl) or b in (0, 16, 31):
            print(b, "nmse first/last", nm[0], nm[-1], "clamped iters", sum(cl), "max alpha", al.max(), "tau min", min(r.tau.min() for r in tr.records))
