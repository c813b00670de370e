"""Debug: attribute fp32 threshold flips in teacher-forced steps (tau vs r perturbation)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import vdamp_oracle as O
from paper_1911_01234_b200 import vdamp, wavelet, workload

w = workload.make_workload("cfg1", batch=1)
p = O.Problem(w.ys[0].astype(np.complex128), w.masks[0].indices, w.pmap.probs, w.noise_vars[0], 4)
lay = wavelet.SubbandLayout.create(256, 256, 4)
rt = np.zeros(65536, dtype=np.complex128)
for k in range(12):
    st = O.step(p, rt)
    g = vdamp.iterate(vdamp.VdampState(wavelet.WaveletCoeffs(rt, lay), k=k), w.ys[0], w.masks[0], w.pmap,
                      w.noise_vars[0], precision="fp32")
    for j, bd in enumerate(p.bands):
        sl = slice(bd.offset, bd.offset + bd.length)
        tg, to = g.thresholds[j], st.thresholds[j]
        if abs(tg - to) > 1e-4 * to:
            mg = np.sort(np.abs(g.r.values[sl].astype(np.complex64)).astype(np.float64))
            mo32 = np.sort(np.abs(st.r[sl].astype(np.complex64)).astype(np.float64))
            t_gpu_data = O.threshold_scan(mg, g.tau.values[j])[0]
            t_o_gtau = O.threshold_scan(np.sort(np.abs(st.r[sl])), g.tau.values[j])[0]
            t_o32 = O.threshold_scan(mo32, st.tau[j])[0]
            print(f"k={k} j={j} n={bd.length} t_gpu={tg:.6g} t_or={to:.6g} scan(gpu r,gpu tau)={t_gpu_data:.6g} "
                  f"scan(or r, gpu tau)={t_o_gtau:.6g} scan(or r c64, or tau)={t_o32:.6g} "
                  f"tau rel={(g.tau.values[j]-st.tau[j])/st.tau[j]:.2e} r rel={np.linalg.norm(g.r.values[sl]-st.r[sl])/np.linalg.norm(st.r[sl]):.2e}")
    rt = st.r_tilde
print("done")
