import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import golden
from oracle import vdamp_oracle as O
from paper_1911_01234_b200 import fourier, vdamp, wavelet, denoise
g = golden("run_full64")
mask = fourier.SamplingMask(g["sampled"])
lay = wavelet.SubbandLayout.create(64, 64, 4)
st = vdamp.iterate(vdamp.initial_state(lay), g["y"], mask, g["probs"], 0.0)
r = st.r.values
tau = np.maximum(st.tau.values, 1e-300)
for rep in range(3):
    st2 = vdamp.iterate(vdamp.initial_state(lay), g["y"], mask, g["probs"], 0.0)
    w2, a2, l2 = denoise.denoise_colored(wavelet.WaveletCoeffs(r, lay), denoise.SubbandVector(tau))
    print(rep, "iterate thr12", st2.thresholds[12], "alpha12", st2.alpha.values[12], "| denoise thr12", l2.values[12]*tau[12], "alpha", a2.values[12])
# scaled problem: same r * 1e10 with tau 1e-280
w3, a3, l3 = denoise.denoise_colored(wavelet.WaveletCoeffs(r * 1e10, lay), denoise.SubbandVector(tau * 1e20))
print("scaled", (l3.values * tau * 1e20)[12], a3.values[12])
t2 = np.full(13, 1e-3)
w4, a4, l4 = denoise.denoise_colored(wavelet.WaveletCoeffs(r, lay), denoise.SubbandVector(t2))
o = O.denoise_colored(r, t2, O.band_table(64, 64, 4))
print("tau=1e-3 gpu", (l4.values*t2)[10:], "oracle", o[3][10:])
