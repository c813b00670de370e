"""FISTA and SURE-IT on the B200 kernels (mirrors src/baselines.py).

Both reuse the VDAMP gradient step (K1 synthesis + row FFT, K2 column
FFT/residual/IFFT, K3 row IFFT + analysis) with unit weights on the mask (no
density compensation, no Onsager), then a fused threshold + momentum update
on the device.  FISTA uses one global threshold per image, SURE-IT the
exact SURE selection of K4 with the oracle error level tau_k = |r_k - w0|^2/N.
``tune_lambda`` runs the whole lambda grid as one batch.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fourier import SamplingMask
from .trace import IterationRecord, RunTrace
from .vdamp import _nmse_db, _subband_nmse
from .wavelet import SubbandLayout, WaveletCoeffs


@dataclass(frozen=True)
class BaselineConfig:
    """src/baselines.py:26-38."""

    algorithm: str
    n_iters: int
    lam: float | None = None

    def __post_init__(self):
        if self.algorithm not in ("fista", "sure_it"):
            raise ValueError(f"unknown baseline algorithm {self.algorithm!r}")
        if self.algorithm == "fista" and (self.lam is None or self.lam <= 0):
            raise ValueError("fista requires lam > 0")
        if self.n_iters < 1:
            raise ValueError("need at least one iteration")


def _setup(plan, ys, mask: SamplingMask, ground_truths):
    n = mask.n
    B = len(ys)
    y = np.concatenate([np.asarray(v) for v in ys])
    idx = np.tile(mask.indices.astype(np.int64), B)
    plan.set_measurements(y, idx, np.full(B, n), np.ones(mask.shape), np.zeros(B), shared_probs=True)
    if ground_truths is not None:
        plan.set_ground_truth(np.stack([np.asarray(g) for g in ground_truths]))


def _run(alg, ys, mask, lams, n_iters, scales, ground_truths, precision, device, want_trace):
    import torch
    from .plan import get_plan
    if n_iters < 1:
        raise ValueError(f"need at least one iteration, got {n_iters}")
    for y in ys:
        if np.shape(y) != (mask.n,):
            raise ValueError(f"measurement length {np.shape(y)} != mask count {mask.n}")
    H, W = mask.shape
    SubbandLayout.create(H, W, scales)
    B = len(ys)
    plan = get_plan(H, W, scales, B, precision, device)
    _setup(plan, ys, mask, ground_truths)
    lam_d = torch.tensor(np.asarray(lams, dtype=np.float64), device=plan.device) if lams is not None else None
    x = plan.empty_images()
    trace = plan.new_trace(n_iters) if want_trace else None
    nmse = (torch.zeros((n_iters, B, 2), dtype=torch.float64, device=plan.device)
            if ground_truths is not None else None)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(_lib.load().vdamp_baseline_run(plan.handle, alg, int(n_iters), _lib.ptr(lam_d), _lib.ptr(x),
                                              _lib.ptr(trace), _lib.ptr(nmse), _lib.stream_ptr()))
    e1.record()
    e1.synchronize()
    wall = e0.elapsed_time(e1) / 1e3 / n_iters
    return (x.cpu().numpy().astype(np.complex128), trace.cpu().numpy() if trace is not None else None,
            nmse.cpu().numpy() if nmse is not None else None, wall)


def fista(y, mask: SamplingMask, lam: float, n_iters: int, scales: int = 4, ground_truth=None,
          *, precision="fp64", device=None):
    """Accelerated soft thresholding with a global threshold (src/baselines.py:54-91)."""
    if lam <= 0:
        raise ValueError(f"lam must be > 0, got {lam}")
    x, tr, nm, wall = _run(0, [y], mask, [lam], n_iters, scales,
                           None if ground_truth is None else [ground_truth], precision, device,
                           ground_truth is not None)
    trace = RunTrace("fista")
    for k in range(n_iters):
        rec = IterationRecord(k=k, wall_time=wall)
        if nm is not None:
            rec.nmse_db = _nmse_db(float(nm[k, 0, 0]), float(nm[k, 0, 1]))
            rec.subband_nmse_db = _subband_nmse(tr[k, 0, :, 6], tr[k, 0, :, 7])
        trace.append(rec)
    return x[0], trace


def sure_it(y, mask: SamplingMask, w0: WaveletCoeffs, n_iters: int, scales: int = 4, ground_truth=None,
            *, precision="fp64", device=None):
    """SURE-tuned thresholding with the oracle scalar error level (src/baselines.py:115-164)."""
    lay = SubbandLayout.create(mask.shape[0], mask.shape[1], scales)
    wl = w0.layout
    if (wl.image_height, wl.image_width, wl.scales) != (lay.image_height, lay.image_width, lay.scales):
        raise ValueError("ground-truth coefficients use a different layout")
    from .wavelet import idwt
    x0 = idwt(WaveletCoeffs(np.asarray(w0.values), lay), precision="fp64")   # the device keeps w0 = dwt(x0)
    x, tr, nm, wall = _run(1, [y], mask, None, n_iters, scales, [x0], precision, device, True)
    trace = RunTrace("sure_it")
    for k in range(n_iters):
        t = tr[k, 0]
        rec = IterationRecord(k=k, wall_time=wall, tau=t[:, 0].copy(), thresholds=t[:, 2] * t[:, 0],
                              lambdas=t[:, 2].copy(), alphas=t[:, 4].copy())
        if ground_truth is not None:
            rec.nmse_db = _nmse_db(float(nm[k, 0, 0]), float(nm[k, 0, 1]))
            rec.subband_nmse_db = _subband_nmse(t[:, 6], t[:, 7])
        trace.append(rec)
    return x[0], trace


def tune_lambda(y, mask: SamplingMask, x0, budget_iters: int, grid, scales: int = 4, *,
                precision="fp64", device=None) -> float:
    """Threshold minimising the NMSE after ``budget_iters`` (src/baselines.py:94-112);
    the whole grid runs as one batch, ties keep the smaller lambda."""
    grid = np.sort(np.asarray(grid, dtype=float))
    if grid.size == 0:
        raise ValueError("empty lambda grid")
    _, _, nm, _ = _run(0, [y] * grid.size, mask, grid, budget_iters, scales, [x0] * grid.size,
                       precision, device, False)
    best, best_nm = None, np.inf
    for b, lam in enumerate(grid):
        s = _nmse_db(float(nm[-1, b, 0]), float(nm[-1, b, 1]))
        if s < best_nm:
            best, best_nm = float(lam), s
    return best
