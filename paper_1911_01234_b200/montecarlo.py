"""Batched Monte Carlo study of the VDAMP state evolution.

Reproduces the reference's 300-mask study (tests/conftest.py:41-81): for each
draw a fresh mask (draw_mask) and noise (synthesize) from the pinned
SeedSequence spawn pairs, the first ``n_iters`` iterates r_k of VDAMP, and the
per-iteration means of r_k, tau_k and the per-subband squared error of r_k
against w0 = dwt(x0).  All draws of a chunk run as one batched
reconstruction on the GPU; the sums are accumulated on the device in a fixed
order (vdamp_mc_accumulate), so the study is deterministic.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .sampling import draw_mask, synthesize
from .wavelet import SubbandLayout


@dataclass
class MonteCarloStudy:
    layout: SubbandLayout
    w0_values: np.ndarray
    mean_r: list = field(default_factory=list)        # per k: (N,) complex
    mean_tau: list = field(default_factory=list)      # per k: (S,)
    mean_sq_err: list = field(default_factory=list)   # per k: (S,)
    n_draws: int = 0
    elapsed: float = 0.0


def draws(pmap, x0, n_draws, seed, snr_db=40.0):
    """(mask, KSpaceData) per draw, exactly as the reference harness spawns them."""
    root = np.random.SeedSequence(seed)
    kids = root.spawn(2 * n_draws)
    for d in range(n_draws):
        mask = draw_mask(pmap, kids[2 * d])
        yield mask, synthesize(x0, mask, snr_db, kids[2 * d + 1])


def mc_study(x0, pmap, n_draws=300, n_iters=3, scales=4, seed=20240801, snr_db=40.0, *,
             chunk=100, precision="fp64", device=None) -> MonteCarloStudy:
    import torch
    from . import _lib
    from .plan import get_plan
    from .vdamp import run_batch
    from .wavelet import dwt
    x0 = np.asarray(x0)
    H, W = x0.shape
    layout = SubbandLayout.create(H, W, scales)
    w0 = dwt(x0, scales, precision="fp64").values
    study = MonteCarloStudy(layout, w0.copy())
    S = layout.n_subbands
    t0 = time.perf_counter()
    gen = draws(pmap, x0, n_draws, seed, snr_db)
    sum_tau = np.zeros((n_iters, S))
    sum_r = sum_sq = scratch = None
    done = 0
    while done < n_draws:
        b = min(chunk, n_draws - done)
        batch = [next(gen) for _ in range(b)]
        masks = [m for m, _ in batch]
        ys = [k.values for _, k in batch]
        nvs = [k.noise_var for _, k in batch]
        _, traces = run_batch(ys, masks, pmap, nvs, scales, n_iters, keep_r_iters=tuple(range(n_iters)),
                              precision=precision, device=device, return_tensor=True, keep_device=True)
        plan = get_plan(H, W, scales, b, precision, device)
        if sum_r is None:
            sum_r = torch.zeros((n_iters, H * W, 2), dtype=torch.float64, device=plan.device)
            sum_sq = torch.zeros((n_iters, S), dtype=torch.float64, device=plan.device)
            scratch = torch.empty(H * W, dtype=torch.float64, device=plan.device)
            w0_d = plan.to_device(w0, plan.cdtype)
        for k in range(n_iters):
            r_k = traces[0].device_snapshots[k]
            _lib.check(_lib.load().vdamp_mc_accumulate(
                plan.handle, _lib.ptr(r_k), _lib.ptr(w0_d), _lib.ptr(sum_r[k]), _lib.ptr(sum_sq[k]),
                _lib.ptr(scratch), _lib.stream_ptr()))
            for tr in traces:
                sum_tau[k] += tr.records[k].tau
        done += b
    torch.cuda.synchronize(plan.device)
    study.elapsed = time.perf_counter() - t0
    study.n_draws = n_draws
    sr = sum_r.cpu().numpy()
    study.mean_r = [(sr[k, :, 0] + 1j * sr[k, :, 1]) / n_draws for k in range(n_iters)]
    study.mean_tau = [sum_tau[k] / n_draws for k in range(n_iters)]
    sq = sum_sq.cpu().numpy()
    study.mean_sq_err = [sq[k] / n_draws for k in range(n_iters)]
    return study
