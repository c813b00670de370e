import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_01234_b200 import vdamp, workload
from oracle import vdamp_oracle as O
w = workload.make_workload("cfg2", batch=32)
rec = vdamp.BatchReconstructor(512, 512, 5, 32, precision="fp32")
inp = vdamp.prepare_batch(w.ys, w.masks, w.pmap, w.noise_vars)
prev = 0.0
for n in (1, 2, 5, 10, 20, 30, 40, 50):
    rec.plan.set_timing(True)
    x = rec(inp.y, inp.indices, inp.counts, inp.probs, inp.noise_var, n)
    kt = rec.plan.kernel_times(); rec.plan.set_timing(False)
    print(n, "select ms", round(kt["sure_select"][0], 2), "launches", kt["sure_select"][1])
