"""CPU-only checks: the C ABI library loads and exports every declared symbol,
argument validation maps to the reference's exceptions, host-side input
generation is pinned to the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def _declared():
    src = open(os.path.join(ROOT, "include", "vdamp_b200.h")).read()
    return sorted(set(re.findall(r"VDAMP_API\s+[\w\s\*]+?\b(vdamp_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_1911_01234_b200 import _lib
    decl = _declared()
    assert len(decl) >= 18
    assert sorted(_lib.SIGNATURES) == decl


def test_library_exports_every_symbol():
    from paper_1911_01234_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.vdamp_abi_version() == 1


def test_plan_create_validation_without_gpu():
    """Shape/scale checks happen before any CUDA call (src/wavelet.py:43-51)."""
    from paper_1911_01234_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.vdamp_plan_create(64, 64, 0, 1, 0, 0, ctypes.byref(h)) == _lib.VDAMP_ERR_ARG
    assert lib.vdamp_plan_create(64, 64, 7, 1, 0, 0, ctypes.byref(h)) == _lib.VDAMP_ERR_SHAPE
    assert lib.vdamp_plan_create(48, 48, 2, 1, 0, 0, ctypes.byref(h)) == _lib.VDAMP_ERR_UNSUPPORTED
    assert lib.vdamp_plan_create(64, 64, 2, 1, 7, 0, ctypes.byref(h)) == _lib.VDAMP_ERR_ARG
    assert lib.vdamp_plan_create(64, 64, 7, 1, 0, 0, ctypes.byref(h)) == _lib.VDAMP_ERR_SHAPE
    assert b"not divisible" in lib.vdamp_last_error()
    with pytest.raises(_lib.DimensionError):
        _lib.check(lib.vdamp_plan_create(64, 64, 7, 1, 0, 0, ctypes.byref(h)))


def test_layout_matches_reference():
    from paper_1911_01234_b200 import DimensionError, SubbandLayout
    ops = golden("operators")
    for key in [k[len("offsets_"):] for k in ops if k.startswith("offsets_")]:
        h, rest = key.split("x")
        w, s = rest.split("s")
        lay = SubbandLayout.create(int(h), int(w), int(s))
        assert [b.offset for b in lay.subbands] == list(ops["offsets_" + key])
    with pytest.raises(DimensionError):
        SubbandLayout.create(64, 64, 7)
    with pytest.raises(ValueError):
        SubbandLayout.create(64, 64, 0)
    lay = SubbandLayout.create(16, 16, 2)
    assert [b.length for b in lay.subbands] == [16, 16, 16, 16, 64, 64, 64]


def test_sampling_pinned_to_reference():
    from paper_1911_01234_b200 import sampling
    g = golden("sampling")
    pm = sampling.polynomial_pmap(64, 48, 8, 0.02, 4.0)
    assert np.array_equal(pm.probs, g["probs_64x48"])
    assert np.array_equal(sampling.draw_mask(pm, 7).sampled, g["mask_64x48_seed7"])
    assert np.array_equal(sampling.polynomial_pmap(96, 96, 6, 0.1, 5.0).probs, g["probs_96_d6"])


def test_baseline_density_and_workload():
    from paper_1911_01234_b200 import workload
    for name in ("cfg1", "cfg2", "cfg3", "cfg4_r2", "cfg4_r16"):
        cfg = workload.CONFIGS[name]
        pm = workload.density(cfg)
        N = cfg.size ** 2
        assert abs(pm.expected_samples() - N / cfg.undersampling) <= 1e-3 * N / cfg.undersampling
        c, h = cfg.size // 2, cfg.centre // 2
        assert np.all(pm.probs[c - h:c + h, c - h:c + h] == 1.0)
    w1 = workload.make_workload("cfg1", batch=2)
    w2 = workload.make_workload("cfg1", batch=1, first=1)
    assert np.array_equal(w1.masks[1].sampled, w2.masks[0].sampled)
    assert np.array_equal(w1.ys[1], w2.ys[0])
    assert w1.ys[0].dtype == np.complex64 and w1.x0.dtype == np.complex64
    assert not np.array_equal(w1.masks[0].sampled, w1.masks[1].sampled)


def test_prepare_batch_validation():
    from paper_1911_01234_b200 import fourier, vdamp
    m = fourier.SamplingMask(np.eye(8, dtype=bool))
    with pytest.raises(ValueError):
        vdamp.prepare_batch([np.zeros(m.n - 1)], [m], np.ones((8, 8)), [0.0])
    with pytest.raises(ValueError):
        vdamp.prepare_batch([np.zeros(m.n)], [m], np.zeros((8, 8)), [0.0])
    with pytest.raises(ValueError):
        vdamp.prepare_batch([np.zeros(m.n)], [m], np.ones((8, 8)), [-1.0])
    inp = vdamp.prepare_batch([np.ones(m.n), 2 * np.ones(m.n)], [m, m], np.ones((8, 8)), [0.1, 0.2])
    assert inp.shared_probs and list(inp.counts) == [8, 8] and inp.indices.size == 16


def test_algorithmic_bytes_formula():
    from paper_1911_01234_b200 import workload
    # 256^2 R4 -> 3,874,816 B (n = N/4)
    assert workload.algorithmic_bytes_per_image_iter(65536, 16384) == 3874816
    assert workload.algorithmic_bytes_per_image_iter(512 * 512, 512 * 512 // 8) == 15106048


def test_check_measurements_c_abi_without_gpu():
    """vdamp_check_measurements (host arrays, no device): a bad index, a repeated index or a
    probability outside (0, 1] is VDAMP_ERR_ARG, as the reference raises ValueError
    (src/fourier.py:65-74, src/sampling.py:45-46); valid inputs pass."""
    from paper_1911_01234_b200 import _lib
    lib = _lib.load()
    H = W = 8
    probs = np.full(H * W, 0.5)
    nv = np.array([0.1, 0.2])

    def call(idx, counts, pr=probs, stride=0, noise=nv):
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        pr = np.ascontiguousarray(pr, dtype=np.float64)
        noise = np.ascontiguousarray(noise, dtype=np.float64)
        P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
        return lib.vdamp_check_measurements(H, W, len(counts), P(idx, ctypes.c_int64), P(counts, ctypes.c_int64),
                                            P(pr, ctypes.c_double), stride, P(noise, ctypes.c_double))

    good = [0, 5, 63, 0, 7]
    assert call(good, [3, 2]) == _lib.VDAMP_OK
    assert call([0, 64, 3, 1, 2], [3, 2]) == _lib.VDAMP_ERR_ARG
    assert b"outside [0" in lib.vdamp_last_error()
    assert call([0, -1, 3, 1, 2], [3, 2]) == _lib.VDAMP_ERR_ARG
    assert call([0, 5, 5, 1, 2], [3, 2]) == _lib.VDAMP_ERR_ARG
    assert b"repeated" in lib.vdamp_last_error()
    bad = probs.copy()
    bad[63] = 0.0
    assert call(good, [3, 2], bad) == _lib.VDAMP_ERR_ARG
    assert b"probability" in lib.vdamp_last_error()
    bad[63] = 1.5
    assert call(good, [3, 2], bad) == _lib.VDAMP_ERR_ARG
    bad[63] = np.nan
    assert call(good, [3, 2], bad) == _lib.VDAMP_ERR_ARG
    assert call(good, [3, 2], np.tile(probs, 2), stride=H * W) == _lib.VDAMP_OK
    assert call(good, [3, 2], stride=5) == _lib.VDAMP_ERR_ARG
    assert call(good, [0, 5]) == _lib.VDAMP_ERR_ARG
    assert call(good, [3, 2], noise=np.array([0.1, -1.0])) == _lib.VDAMP_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(call([0, 64, 3, 1, 2], [3, 2]))
