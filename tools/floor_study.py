"""complex64-floor study on the BASELINE workloads, CPU only.

For each config and slice: the oracle in float64 vs the oracle with its state
rounded to complex64 every iteration (oracle.run(c64_state=True)); prints the
final x_hat rel-L2 and the max per-iteration |dNMSE|.  Builder tooling.
"""
import json
import multiprocessing as mp
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(args):
    from oracle import vdamp_oracle as O
    from paper_1911_01234_b200 import workload
    name, b = args
    w = workload.make_workload(name, batch=1, first=b)
    cfg = w.config
    a = dict(ground_truth=w.x0[0].astype(np.complex128))
    ref = O.run(w.ys[0].astype(np.complex128), w.masks[0].indices, w.pmap.probs, w.noise_vars[0], cfg.scales,
                cfg.n_iters, **a)
    flo = O.run(w.ys[0].astype(np.complex128), w.masks[0].indices, w.pmap.probs, w.noise_vars[0], cfg.scales,
                cfg.n_iters, c64_state=True, **a)
    rel = float(np.linalg.norm(flo.x_hat - ref.x_hat) / np.linalg.norm(ref.x_hat))
    dn = float(max(abs(x.nmse_db - y.nmse_db) for x, y in zip(flo.records, ref.records)))
    return name, b, rel, dn, ref.records[-1].nmse_db


if __name__ == "__main__":
    jobs = []
    spec = dict(cfg1=range(4), cfg2=range(4), cfg3=range(1), cfg4_r2=range(4), cfg4_r8=range(4), cfg4_r16=range(4))
    if len(sys.argv) > 1:
        spec = {k: v for k, v in spec.items() if k in sys.argv[1:]}
    for k, r in spec.items():
        jobs += [(k, b) for b in r]
    with mp.Pool(min(len(jobs), os.cpu_count())) as pool:
        for res in pool.imap_unordered(one, jobs):
            print(json.dumps(dict(zip(("config", "slice", "rel_l2", "max_dnmse_db", "final_nmse_db"), res))), flush=True)
