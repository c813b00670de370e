import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_01234_b200 import vdamp, workload
cfg, b, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
w = workload.make_workload(cfg, batch=b)
x, _ = vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, w.config.scales, 3, precision=prec)
print("ok", cfg, b, prec, np.isfinite(x).all())
