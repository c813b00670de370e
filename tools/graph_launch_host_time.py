"""Host time of one vdamp_run call (graph replay) on cfg1, device-resident inputs: how long the
launching thread is busy per batch (the streaming API pipelines batches, so this bounds its rate)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_01234_b200 import vdamp, workload
w = workload.make_workload("cfg1", procs=8)
inp = vdamp.prepare_batch(w.ys, w.masks, w.pmap, w.noise_vars)
rec = vdamp.BatchReconstructor(256, 256, 4, 64, precision="fp32")
dev = rec.plan.device
y = torch.from_numpy(inp.y).to(dev, rec.plan.cdtype); idx = torch.from_numpy(inp.indices).to(dev); pr = torch.from_numpy(inp.probs).to(dev)
for _ in range(3):
    rec(y, idx, inp.counts, pr, inp.noise_var, 30, sync=True)
ts = []
t_all = time.perf_counter()
for _ in range(20):
    t0 = time.perf_counter()
    rec(y, idx, inp.counts, pr, inp.noise_var, 30, sync=False)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
t_all = time.perf_counter() - t_all
print("host ms per call: median %.3f max %.3f; wall per call %.3f ms" % (1e3 * np.median(ts), 1e3 * max(ts), 1e3 * t_all / 20))
