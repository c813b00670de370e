"""Sanity of the large-geometry paths (2048^2, 1024 x 2048, 2048 x 512): fp32 against fp64 on the GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_01234_b200 import vdamp, sampling
from paper_1911_01234_b200.plan import clear_plans

for (h, w, s) in [(2048, 2048, 2), (1024, 2048, 3), (2048, 512, 4), (512, 1024, 1)]:
    rng = np.random.default_rng(5)
    x0 = (rng.standard_normal((h, w)) * (rng.random((h, w)) < 0.05)).astype(np.complex128)
    pmap = sampling.polynomial_pmap(h, w, undersampling=4.0)
    mask = sampling.draw_mask(pmap, 1)
    kd = sampling.synthesize(x0, mask, 35.0, 2)
    x64, _ = vdamp.run(kd.values, mask, pmap, kd.noise_var, s, 4, precision="fp64")
    x32, _ = vdamp.run(kd.values, mask, pmap, kd.noise_var, s, 4, precision="fp32")
    rel = np.linalg.norm(x32 - x64) / np.linalg.norm(x64)
    print(h, w, s, "fp32 vs fp64 rel", rel, flush=True)
    assert np.isfinite(rel) and rel < 3e-2, rel
    clear_plans()
print("ok")
