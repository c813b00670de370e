import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import golden
from oracle import vdamp_oracle as O
from paper_1911_01234_b200 import fourier, vdamp, wavelet
g = golden("run_full64")
mask = fourier.SamplingMask(g["sampled"])
lay = wavelet.SubbandLayout.create(64, 64, 4)
st = vdamp.iterate(vdamp.initial_state(lay), g["y"], mask, g["probs"], 0.0)
b = lay.subbands[12]
seg = st.r.values[b.offset:b.offset+b.length]
m = np.sort(np.abs(seg)); n = m.size; tau = 1e-300
np.save("/root/repo/gpurun_out/seg12.npy", seg)
print("oracle scan", O.threshold_scan(m, tau))
for t in (0.0, 1.387914615456682e-16):
    print("sure_risk", t, O.sure_risk(seg, tau, t))
