"""Experiment: split a cfg1 batch into k independent plans on k streams (device-resident timing).

usage: python tools/exp_streams.py [k] [steps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_01234_b200 import vdamp, workload
from paper_1911_01234_b200.plan import Plan

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = workload.CONFIGS["cfg1"]
B = cfg.batch
w = workload.make_workload("cfg1")
per = B // k
dev = torch.device("cuda", 0)
lanes = []
for i in range(k):
    sl = slice(i * per, (i + 1) * per)
    inp = vdamp.prepare_batch(w.ys[sl], w.masks[sl], w.pmap, w.noise_vars[sl])
    plan = Plan(cfg.size, cfg.size, cfg.scales, per, "fp32", 0)
    st = torch.cuda.Stream(dev)
    d = dict(y=torch.from_numpy(inp.y).to(dev, plan.cdtype), idx=torch.from_numpy(inp.indices).to(dev),
             counts=inp.counts, probs=torch.from_numpy(inp.probs).to(dev), nv=inp.noise_var)
    lanes.append((plan, st, d, plan.empty_images()))

def step():
    for plan, st, d, x in lanes:
        with torch.cuda.stream(st):
            plan.set_measurements(d["y"], d["idx"], d["counts"], d["probs"], d["nv"], True, stream=st)
            plan.run(cfg.n_iters, x_hat=x, stream=st)

for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
main = torch.cuda.current_stream()
e0.record(main)
for s_ in [l[1] for l in lanes]:
    s_.wait_stream(main)
for _ in range(steps):
    step()
for s_ in [l[1] for l in lanes]:
    main.wait_stream(s_)
e1.record(main)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"k={k}: {B * cfg.n_iters / (ms / 1e3):.0f} img-iter/s ({ms:.3f} ms/step)")
