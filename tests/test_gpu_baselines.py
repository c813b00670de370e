"""FISTA / SURE-IT / tune_lambda on the GPU vs fixtures of src/baselines.py."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rel2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_fista_vs_reference():
    from paper_1911_01234_b200 import baselines
    from paper_1911_01234_b200.fourier import SamplingMask
    g = golden("baselines")
    x, tr = baselines.fista(g["y"], SamplingMask(g["sampled"]), 0.01, 12, 4, ground_truth=g["x0"])
    assert rel2(x, g["fista_x"]) <= 1e-9
    assert np.abs(tr.nmse_curve() - g["fista_nmse"]).max() <= 1e-6
    sb = np.array([r.subband_nmse_db for r in tr.records])
    assert np.allclose(sb, g["fista_sbn"], atol=1e-6, equal_nan=True)


def test_sure_it_vs_reference():
    from paper_1911_01234_b200 import baselines, wavelet
    from paper_1911_01234_b200.fourier import SamplingMask
    g = golden("baselines")
    w0 = wavelet.dwt(g["x0"], 4)
    x, tr = baselines.sure_it(g["y"], SamplingMask(g["sampled"]), w0, 10, 4, ground_truth=g["x0"])
    assert rel2(x, g["sure_x"]) <= 1e-8
    assert np.allclose(np.array([r.tau for r in tr.records]), g["sure_tau"], rtol=1e-9)
    assert np.allclose(np.array([r.thresholds for r in tr.records]), g["sure_thr"], rtol=1e-8)
    assert np.abs(tr.nmse_curve() - g["sure_nmse"]).max() <= 1e-6
    sb = np.array([r.subband_nmse_db for r in tr.records])
    assert np.allclose(sb, g["sure_sbn"], atol=1e-6, equal_nan=True)


def test_tune_lambda_vs_reference():
    from paper_1911_01234_b200 import baselines
    from paper_1911_01234_b200.fourier import SamplingMask
    g = golden("baselines")
    lam = baselines.tune_lambda(g["y"], SamplingMask(g["sampled"]), g["x0"], 8, g["grid"], 4)
    assert lam == float(g["lam"])


def test_baseline_config_validation():
    from paper_1911_01234_b200.baselines import BaselineConfig
    with pytest.raises(ValueError):
        BaselineConfig("fista", 10)
    with pytest.raises(ValueError):
        BaselineConfig("nope", 10, 1.0)
    BaselineConfig("sure_it", 5)
