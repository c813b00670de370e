"""Where does the fp32 path leave the float64 oracle?  Teacher-forced along the oracle's own
trajectory: at every iteration the fp32 GPU step from the oracle's r~_k, compared per subband
(r, tau, threshold); a threshold that differs is classified by the oracle's exact SURE risk at
both thresholds (near-tie = relative risk excess <= 1e-6) and by the relative gap.
Usage: python tools/fp32_divergence.py cfg2 0 [n_iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import vdamp_oracle as O  # noqa: E402
from paper_1911_01234_b200 import vdamp, wavelet, workload  # noqa: E402

name, b = sys.argv[1], int(sys.argv[2])
w = workload.make_workload(name, batch=1, first=b)
c = w.config
K = int(sys.argv[3]) if len(sys.argv) > 3 else c.n_iters
p = O.Problem(w.ys[0].astype(np.complex128), w.masks[0].indices, w.pmap.probs, w.noise_vars[0], c.scales)
lay = wavelet.SubbandLayout.create(c.size, c.size, c.scales)
rt = np.zeros(c.size * c.size, dtype=np.complex128)
for k in range(K):
    st = O.step(p, rt)
    g = vdamp.iterate(vdamp.VdampState(wavelet.WaveletCoeffs(rt, lay), k=k), w.ys[0], w.masks[0], w.pmap,
                      w.noise_vars[0], precision="fp32")
    rr = np.linalg.norm(g.r.values - st.r) / np.linalg.norm(st.r)
    taur = np.abs(g.tau.values - st.tau) / st.tau
    line = f"k={k:2d} r_rel={rr:.2e} tau_rel_max={taur.max():.2e}"
    for j, bd in enumerate(p.bands):
        sl = slice(bd.offset, bd.offset + bd.length)
        tg, to = g.thresholds[j], st.thresholds[j]
        if abs(tg - to) > 1e-5 * max(to, 1e-30):
            seg = st.r[sl]
            tau = max(st.tau[j], 1e-300)
            rg, ro = O.sure_risk(seg, tau, tg), O.sure_risk(seg, tau, to)
            mg = np.sort(np.abs(g.r.values[sl].astype(np.complex64)).astype(np.float64))
            own = O.threshold_scan(mg, g.tau.values[j])[0]
            line += (f"\n   j={j:2d} n={bd.length} t_gpu={tg:.6g} t_or={to:.6g} dt={(tg-to)/to:+.2e} "
                     f"risk excess={(rg-ro)/abs(ro):.2e} own-data exact scan={own:.6g} "
                     f"tau_rel={taur[j]:.1e}")
    print(line, flush=True)
    rt = st.r_tilde
