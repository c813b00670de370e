"""Artifact writers and experiment config vs the reference CLI's own files
(tests/golden/cli.npz, written by src/cli.py:run_experiment)."""

import csv
import io
import json

import numpy as np
import pytest

from conftest import golden
from paper_1911_01234_b200 import artifacts, experiment
from paper_1911_01234_b200.trace import IterationRecord, RunTrace


def _parse_trace(text):
    rows = list(csv.reader(io.StringIO(text)))[1:]
    run_id = rows[0][0]
    recs = {}
    for _, k, metric, j, _, v in rows:
        k, j, v = int(k), int(j), float(v)
        rec = recs.setdefault(k, {"k": k})
        if j < 0:
            rec[metric] = v
        else:
            rec.setdefault(metric, []).append(v)
    names = {"subband_nmse_db": "subband_nmse_db", "tau": "tau", "threshold": "thresholds",
             "lambda": "lambdas", "alpha": "alphas"}
    tr = RunTrace(run_id.split("_R")[0])
    for k in sorted(recs):
        r = recs[k]
        rec = IterationRecord(k=k, wall_time=r["wall_time"], nmse_db=r.get("nmse_db"))
        for m, f in names.items():
            if m in r:
                setattr(rec, f, np.array(r[m]))
        tr.append(rec)
    return run_id, tr


def test_trace_csv_bytes(tmp_path):
    g = golden("cli")
    for f in g["files"]:
        f = str(f)
        if not f.startswith("trace_"):
            continue
        text = str(g["txt:" + f])
        run_id, tr = _parse_trace(text)
        artifacts.write_trace_csv(tmp_path / f, run_id, tr)
        assert (tmp_path / f).read_text() == text, f


def test_qq_csv_bytes(tmp_path):
    g = golden("cli")
    for f in g["files"]:
        f = str(f)
        if not f.startswith("qq_"):
            continue
        text = str(g["txt:" + f])
        rows = list(csv.reader(io.StringIO(text)))[1:]
        groups = {}
        for run_id, k, j, comp, qt, qe in rows:
            groups.setdefault((int(k), int(j), comp), []).append((float(qt), float(qe)))
        entries = [(k, j, artifacts.QQData(c, np.array([a for a, _ in v]), np.array([b for _, b in v]), 0.0))
                   for (k, j, c), v in groups.items()]
        artifacts.write_qq_csv(tmp_path / f, rows[0][0], entries)
        assert (tmp_path / f).read_text() == text
        # theoretical quantiles: the restated inverse CDF reproduces them exactly
        for (k, j, c), v in groups.items():
            nq = len(v)
            pos = (np.arange(1, nq + 1) - 0.5) / nq
            assert np.array_equal(artifacts.normal_quantile(pos), np.array([a for a, _ in v]))


def test_sidecars_bytes(tmp_path):
    g = golden("cli")
    for f in g["files"]:
        f = str(f)
        if not f.endswith(".bin"):
            continue
        side = json.loads(str(g["txt:" + f + ".json"]))
        arr = g["bin:" + f]
        artifacts.save_array(tmp_path / f, arr, side.get("metadata"))
        assert (tmp_path / (f + ".json")).read_text() == str(g["txt:" + f + ".json"])
        back, meta = artifacts.load_array(tmp_path / f)
        assert back.dtype == arr.dtype and np.array_equal(back, arr) and meta == side.get("metadata", {})


def test_qq_data_statistics():
    rng = np.random.default_rng(3)
    res = rng.normal(size=500) + 1j * rng.normal(size=500)
    re, im = artifacts.qq_data(res, 50)
    assert re.component == "real" and im.component == "imag"
    assert re.correlation > 0.98 and im.correlation > 0.98
    with pytest.raises(ValueError):
        artifacts.qq_data(res[:5], 10)
    with pytest.raises(ValueError):
        artifacts.qq_data(res, 5)


def test_mosaic_layout():
    from paper_1911_01234_b200.wavelet import SubbandLayout
    lay = SubbandLayout.create(16, 8, 2)
    vals = np.arange(128, dtype=float)
    m = artifacts.coeff_mosaic(vals, lay)
    b = lay.subbands[1]                 # horizontal, coarsest: top-right of the corner block
    h, w = b.shape
    assert np.array_equal(m[0:h, w:2 * w].ravel(), vals[b.offset:b.offset + b.length])
    assert sorted(m.ravel()) == list(vals)


def test_config_and_validation(tmp_path):
    g = golden("cli")
    raw = json.loads(str(g["config_json"]))
    cfg = experiment.config_from_dict(raw)
    assert cfg.validate() == []
    man = json.loads(str(g["txt:manifest.json"]))
    assert cfg.to_dict() == man["config"]
    bad = experiment.config_from_dict({"phantom_size": 8, "scales": 0, "undersampling": [0.5],
                                       "density": {"p_min": 0}, "snr_db": -1,
                                       "algorithms": {"fista": {"n_iters": 0}, "x": {}}})
    msgs = bad.validate()
    assert "phantom_size 8 below minimum 16" in msgs
    assert "scales must be >= 1, got 0" in msgs
    assert "fista: needs lam or lambda_grid" in msgs
    assert "unknown algorithm 'x'" in msgs
    with pytest.raises(experiment.ConfigError):
        experiment.config_from_dict({"nonsense": 1})
    p = tmp_path / "c.yaml"
    p.write_text("phantom_size: 32\nscales: 3\n")
    assert experiment.main(["validate", "--config", str(p)]) == 0
    p.write_text("phantom_size: 30\nscales: 3\n")
    assert experiment.main(["validate", "--config", str(p)]) == 2
    p.write_text("[1, 2]\n")
    assert experiment.main(["validate", "--config", str(p)]) == 2
