"""the experiment runner on the GPU writes the reference
CLI's artifacts (tests/golden/cli.npz, from src/cli.py:run_experiment)."""

import csv
import io
import json

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


def test_experiment_matches_reference_cli(tmp_path):
    import yaml
    from paper_1911_01234_b200 import artifacts, experiment
    g = golden("cli")
    cfgp = tmp_path / "exp.yaml"
    cfgp.write_text(yaml.safe_dump(json.loads(str(g["config_json"])), sort_keys=False))
    out = tmp_path / "out"
    assert experiment.main(["run", "--config", str(cfgp), "--out", str(out), "--device", "cuda"]) == 0
    files = sorted(p.name for p in out.iterdir())
    assert files == [str(f) for f in g["files"]]
    for f in files:
        if f.endswith(".bin"):
            ours, _ = artifacts.load_array(out / f)
            ref = g["bin:" + f]
            assert ours.dtype == ref.dtype and ours.shape == ref.shape, f
            if f.startswith(("phantom", "pmap", "mask")):
                assert np.array_equal(ours, ref), f
            else:
                assert np.linalg.norm(ours - ref) <= 1e-8 * np.linalg.norm(ref), f
        elif f.endswith(".bin.json"):
            assert (out / f).read_text() == str(g["txt:" + f]), f
        elif f.endswith(".csv"):
            a, b = _rows((out / f).read_text()), _rows(str(g["txt:" + f]))
            assert len(a) == len(b) and a[0] == b[0], f
            valcol = {"trace": [5], "qq": [4, 5], "subbands": [4]}[f.split("_")[0]]
            for ra, rb in zip(a[1:], b[1:]):
                keys = [i for i in range(len(ra)) if i not in valcol]
                assert [ra[i] for i in keys] == [rb[i] for i in keys], (f, ra, rb)
                if f.startswith("trace") and ra[2] == "wall_time":
                    continue
                for i in valcol:
                    x, y = float(ra[i]), float(rb[i])
                    assert (np.isnan(x) and np.isnan(y)) or abs(x - y) <= 1e-6 * max(1.0, abs(y)), (f, ra, rb)
    man = json.loads((out / "manifest.json").read_text())
    ref = json.loads(str(g["txt:manifest.json"]))
    for k in ("config", "config_sha256", "seed", "substreams"):
        assert man[k] == ref[k]
    assert len(man["cells"]) == len(ref["cells"])
    for a, b in zip(man["cells"], ref["cells"]):
        assert set(a) == set(b)
        for k in ("algorithm", "undersampling", "n_iters", "lam"):
            assert a.get(k) == b.get(k)
        assert abs(a["final_nmse_db"] - b["final_nmse_db"]) <= 1e-6
    assert experiment.main(["list-outputs", "--out", str(tmp_path)]) == 0
