"""Batched Monte Carlo study on the GPU vs the oracle (reference tests/conftest.py:41-81)
and the reference's acceptance criteria 2-3 (tests/test_acceptance.py:63-104)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _oracle_mc(O, x0, pmap, n_draws, n_iters, scales, seed):
    from paper_1911_01234_b200.montecarlo import draws
    bands = O.band_table(*x0.shape, scales)
    w0 = O.dwt(x0, scales)
    lengths = np.array([b.length for b in bands])
    offs = np.concatenate(([0], np.cumsum(lengths)))
    sr = [np.zeros(x0.size, complex) for _ in range(n_iters)]
    st = [np.zeros(len(bands)) for _ in range(n_iters)]
    sq = [np.zeros(len(bands)) for _ in range(n_iters)]
    for mask, k in draws(pmap, x0, n_draws, seed):
        p = O.Problem(k.values, mask.indices, pmap.probs, k.noise_var, scales)
        rt = np.zeros(x0.size, complex)
        for it in range(n_iters):
            s = O.step(p, rt)
            sr[it] += s.r
            st[it] += s.tau
            sq[it] += np.add.reduceat(np.abs(s.r - w0) ** 2, offs[:-1]) / lengths
            rt = s.r_tilde
    return [v / n_draws for v in sr], [v / n_draws for v in st], [v / n_draws for v in sq]


def test_mc_study_matches_oracle_and_acceptance(oracle):
    from paper_1911_01234_b200 import montecarlo, sampling
    x0 = golden("run_shepp128")["x0"]
    pmap = sampling.polynomial_pmap(128, 128, 8, 0.02, 8.0)
    n_draws, seed = 300, 20240801
    study = montecarlo.mc_study(x0, pmap, n_draws=n_draws, n_iters=3, scales=4, seed=seed, chunk=128)
    mr, mt, ms = _oracle_mc(oracle, x0, pmap, n_draws, 3, 4, seed)
    for k in range(3):
        assert np.allclose(study.mean_tau[k], mt[k], rtol=1e-9)
        assert np.allclose(study.mean_sq_err[k], ms[k], rtol=1e-8)
        assert np.abs(study.mean_r[k] - mr[k]).max() <= 1e-9 * np.abs(mr[k]).max()
    # acceptance 2: density-compensated r0 is unbiased (projected bias <= 1%)
    w0 = study.w0_values
    worst = 0.0
    for b in study.layout.subbands:
        sl = slice(b.offset, b.offset + b.length)
        d = float(np.vdot(w0[sl], w0[sl]).real)
        worst = max(worst, abs(np.vdot(w0[sl], study.mean_r[0][sl] - w0[sl]).real / d))
    assert worst <= 0.01
    # acceptance 3: tau tracks the true per-subband error (5% at k=0, 10% after)
    for k, lim in enumerate((0.05, 0.10, 0.10)):
        rel = np.abs(study.mean_tau[k] - study.mean_sq_err[k]) / study.mean_sq_err[k]
        assert rel.max() <= lim, (k, rel.max())
