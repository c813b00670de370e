"""Seeded synthetic workloads of BASELINE.json ``configs`` (no dataset involved).

Every slice b uses ``SeedSequence(entropy=seed, spawn_key=(b, role))`` with
role 0 = phantom, 1 = mask, 2 = noise (the substream style of
src/cli.py:32-33).  Phantoms are random ellipses times a smooth phase,
rounded to complex64; measurements are synthesised in float64 from that
and rounded to complex64, so the GPU path and the CPU oracle see identical
inputs.  The density follows the reference offset law with degree 6 and a
square fully sampled centre (SURVEY finding 4).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sampling import (ProbabilityMap, draw_mask, polynomial_pmap, random_ellipse_phantom,
                       smooth_phase, synthesize)

DEFAULT_SEED = 20261020


@dataclass(frozen=True)
class Config:
    name: str
    batch: int
    size: int
    ellipses: int
    scales: int
    undersampling: float
    centre: int
    snr_db: float
    n_iters: int


CONFIGS = {
    "cfg0": Config("cfg0", 1, 256, 12, 4, 4.0, 24, 40.0, 30),
    "cfg1": Config("cfg1", 64, 256, 12, 4, 4.0, 24, 40.0, 30),
    "cfg2": Config("cfg2", 32, 512, 20, 5, 8.0, 32, 30.0, 50),
    "cfg3": Config("cfg3", 1, 1024, 40, 6, 6.0, 48, 35.0, 50),
    "cfg4_r2": Config("cfg4_r2", 1024, 256, 12, 4, 2.0, 24, 40.0, 30),
    "cfg4_r4": Config("cfg4_r4", 1024, 256, 12, 4, 4.0, 24, 40.0, 30),
    "cfg4_r8": Config("cfg4_r8", 1024, 256, 12, 4, 8.0, 24, 40.0, 30),
    "cfg4_r16": Config("cfg4_r16", 1024, 256, 12, 4, 16.0, 24, 40.0, 30),
}


@dataclass
class Workload:
    config: Config
    pmap: ProbabilityMap
    masks: list
    ys: list            # complex64 measurement vectors
    noise_vars: np.ndarray
    x0: np.ndarray      # (B, H, W) complex64 ground truth
    slices: list = field(default_factory=list)

    @property
    def n_total(self) -> int:
        return int(sum(m.n for m in self.masks))


def density(cfg: Config) -> ProbabilityMap:
    return polynomial_pmap(cfg.size, cfg.size, degree=6, center_radius=0.0,
                           undersampling=cfg.undersampling, p_min=1e-3, center_square=cfg.centre)


def make_slice(cfg: Config, pmap: ProbabilityMap, b: int, seed: int = DEFAULT_SEED):
    ss = lambda role: np.random.SeedSequence(entropy=seed, spawn_key=(b, role))
    rng = np.random.default_rng(ss(0))
    img = random_ellipse_phantom(cfg.size, cfg.size, cfg.ellipses, rng)
    x0 = (img * smooth_phase(cfg.size, cfg.size, rng)).astype(np.complex64)
    mask = draw_mask(pmap, ss(1))
    k = synthesize(x0.astype(np.complex128), mask, cfg.snr_db, ss(2))
    return x0, mask, k.values.astype(np.complex64), float(k.noise_var)


_JOB = None          # (cfg, pmap, seed) of the pool in flight (inherited by the forked workers)


def _slice_job(b):
    cfg, pmap, seed = _JOB
    return make_slice(cfg, pmap, b, seed)


def make_workload(name_or_cfg, batch: int | None = None, seed: int = DEFAULT_SEED, first: int = 0,
                  procs: int = 1) -> Workload:
    """Slices [first, first + batch) of a configuration (default: the whole batch).
    ``procs`` > 1 generates the slices in that many forked processes (same result)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    n = cfg.batch if batch is None else int(batch)
    pmap = density(cfg)
    global _JOB
    _JOB = (cfg, pmap, seed)
    jobs = list(range(first, first + n))
    if procs > 1 and n > 8:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(min(procs, n)) as pool:
            res = pool.map(_slice_job, jobs, chunksize=max(1, n // (4 * procs)))
    else:
        res = [_slice_job(j) for j in jobs]
    xs, masks, ys, nvs = (list(v) for v in zip(*res))
    return Workload(cfg, pmap, masks, ys, np.array(nvs), np.stack(xs), list(range(first, first + n)))


def algorithmic_bytes_per_image_iter(N: int, n: int, complex_bytes: int = 8) -> float:
    """B_iter = 56 N b_c/8 + 12 n b_c/8 + N/8 (3-pass pipeline)."""
    return 56.0 * N * complex_bytes / 8 + 12.0 * n * complex_bytes / 8 + N / 8.0
