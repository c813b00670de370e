"""Experiment: where the streaming e2e time goes (cfg1).  python tools/exp_e2e.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_01234_b200 import vdamp, workload
cfg = workload.CONFIGS["cfg1"]
w = workload.make_workload("cfg1")
inp = vdamp.prepare_batch(w.ys, w.masks, w.pmap, w.noise_vars)
B, S = cfg.batch, 10
srec = vdamp.StreamingReconstructor(cfg.size, cfg.size, cfg.scales, B, precision="fp32")
host = srec.upload(inp, pin=True)
outs = [torch.empty((B, cfg.size, cfg.size), dtype=torch.complex64).pin_memory() for _ in range(2)]
dev = srec.plan.device
dhost = {k: (v.to(dev) if torch.is_tensor(v) else v) for k, v in host.items()}

def timeit(label, fn):
    for i in range(3):
        fn(i)
    srec.wait(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(S):
        fn(i)
    srec.wait(); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / S
    print(f"{label:40s} {dt * 1e3:7.3f} ms/step  {B * cfg.n_iters / dt:9.0f} img-iter/s", flush=True)

timeit("streaming, pinned host in/out", lambda i: srec.submit(host, cfg.n_iters, outs[i & 1]))
dout = [srec.plan.empty_images() for _ in range(2)]
timeit("streaming, device in, device out", lambda i: srec.submit(dhost, cfg.n_iters, dout[i & 1]))
timeit("streaming, pinned in, device out", lambda i: srec.submit(host, cfg.n_iters, dout[i & 1]))
p = srec.plan
st = torch.cuda.Stream(dev)
x = p.empty_images()
def plain(i):
    with torch.cuda.stream(st):
        p.set_measurements(dhost["y"], dhost["indices"], host["counts"], dhost["probs"], host["noise_var"], True, stream=st)
        p.run(cfg.n_iters, x_hat=x, stream=st)
timeit("plan calls only (device inputs)", plain)
t0 = time.perf_counter()
for i in range(S):
    plain(i)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue time per step {1e3 * (t1 - t0) / S:.3f} ms")
