"""Small VDAMP runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the 256-point kernels (fp32 + fp64), the generic kernels (64^2), the 512-point kernels, the
large-subband SURE paths (single-CTA global sort fp64, multi-CTA value ranges fp32) and the
measurement guards.  Builder tooling: tools/sanitize.sh runs it under each tool."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_01234_b200 import denoise, vdamp, wavelet, workload  # noqa: E402

which = sys.argv[1:] or ["256", "64", "512", "sure1024"]
if "256" in which:
    w = workload.make_workload("cfg1", batch=2)
    for prec in ("fp32", "fp64"):
        vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 4, 2, ground_truths=w.x0, precision=prec)
if "64" in which:
    cfg = workload.Config("s64", 2, 64, 6, 3, 4.0, 8, 40.0, 2)
    w = workload.make_workload(cfg)
    for prec in ("fp32", "fp64"):
        vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 3, 2, ground_truths=w.x0, precision=prec)
if "512" in which:
    w = workload.make_workload("cfg2", batch=1)
    vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 5, 1, precision="fp32")
if "sure1024" in which:
    rng = np.random.default_rng(1)
    lay = wavelet.SubbandLayout.create(1024, 1024, 1)
    r = (rng.normal(size=1 << 20) + 1j * rng.normal(size=1 << 20)).astype(np.complex64).astype(np.complex128)
    tau = np.full(lay.n_subbands, 0.5)
    for prec in ("fp32", "fp64"):
        denoise.denoise_colored(wavelet.WaveletCoeffs(r, lay), denoise.SubbandVector(tau), precision=prec)
print("sanitize case done", which)
