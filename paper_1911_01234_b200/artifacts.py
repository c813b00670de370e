"""Experiment artifacts in the reference's on-disk formats.

Restates src/io.py:14-79 (raw little-endian ``.bin`` + JSON sidecar, long-format
trace and QQ CSVs), src/cli.py:94-101 (subband table), src/wavelet.py:151-166
(coefficient mosaic) and src/diagnostics.py:54-149 (QQ quantile pairs) so the
GPU runs write byte-compatible files.  Host-side post-processing only.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .trace import RunTrace

TRACE_COLUMNS = ("run_id", "iter", "metric", "subband", "component", "value")
QQ_COLUMNS = ("run_id", "iter", "subband", "component", "q_theory", "q_emp")


def save_array(path, arr: np.ndarray, metadata: dict | None = None) -> None:
    """Raw C-order dump plus ``<name>.json`` sidecar (src/io.py:18-33)."""
    path = Path(path)
    arr = np.ascontiguousarray(arr)
    arr.tofile(path)
    side = {"dtype": str(arr.dtype), "shape": list(arr.shape), "order": "C"}
    if metadata:
        side["metadata"] = metadata
    path.with_suffix(path.suffix + ".json").write_text(json.dumps(side, indent=2, sort_keys=True) + "\n")


def load_array(path) -> tuple[np.ndarray, dict]:
    """Inverse of :func:`save_array` (src/io.py:36-41)."""
    path = Path(path)
    side = json.loads(path.with_suffix(path.suffix + ".json").read_text())
    arr = np.fromfile(path, dtype=np.dtype(side["dtype"])).reshape(side["shape"])
    return arr, side.get("metadata", {})


def _fmt(v) -> str:
    return repr(float(v))


def trace_rows(run_id: str, trace: RunTrace):
    """Rows of the long-format trace table, subband -1 = whole image (src/io.py:48-72)."""
    for rec in trace.records:
        yield (run_id, rec.k, "wall_time", -1, "", _fmt(rec.wall_time))
        if rec.nmse_db is not None:
            yield (run_id, rec.k, "nmse_db", -1, "", _fmt(rec.nmse_db))
        for metric, vals in (("subband_nmse_db", rec.subband_nmse_db), ("tau", rec.tau),
                             ("threshold", rec.thresholds), ("lambda", rec.lambdas), ("alpha", rec.alphas)):
            if vals is None:
                continue
            for j, v in enumerate(vals):
                yield (run_id, rec.k, metric, j, "", _fmt(v))


def write_trace_csv(path, run_id: str, trace: RunTrace) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_COLUMNS)
        w.writerows(trace_rows(run_id, trace))


def write_qq_csv(path, run_id: str, entries) -> None:
    """entries: (iteration, subband, QQData) (src/io.py:75-82)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(QQ_COLUMNS)
        for k, j, qq in entries:
            for a, b in zip(qq.q_theory, qq.q_empirical):
                w.writerow((run_id, k, j, qq.component, _fmt(a), _fmt(b)))


def write_subband_csv(path, layout, energies) -> None:
    """Per-subband ground-truth energy table (src/cli.py:94-101)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(("subband", "scale", "orientation", "length", "w0_energy"))
        for j, b in enumerate(layout.subbands):
            w.writerow((j, b.scale, b.orientation, b.length, repr(float(energies[j]))))


_QUADRANT = {"approx": (0, 0), "horizontal": (0, 1), "vertical": (1, 0), "diagonal": (1, 1)}


def coeff_mosaic(values: np.ndarray, layout) -> np.ndarray:
    """Nested 2D arrangement of the flat coefficients (src/wavelet.py:151-166)."""
    out = np.empty((layout.image_height, layout.image_width), dtype=values.dtype)
    for b in layout.subbands:
        h, w = b.shape
        qi, qj = _QUADRANT[b.orientation]
        out[qi * h:(qi + 1) * h, qj * w:(qj + 1) * w] = values[b.offset:b.offset + b.length].reshape(h, w)
    return out


# Acklam's rational approximation of the standard normal inverse CDF (the
# published coefficients; src/diagnostics.py:54-110 uses the same method)
_A = (-3.969683028665376e01, 2.209460984245205e02, -2.759285104469687e02,
      1.383577518672690e02, -3.066479806614716e01, 2.506628277459239e00)
_B = (-5.447609879822406e01, 1.615858368580409e02, -1.556989798598866e02,
      6.680131188771972e01, -1.328068155288572e01, 1.0)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e00,
      -2.549732539343734e00, 4.374664141464968e00, 2.938163982698783e00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e00,
      3.754408661907416e00, 1.0)
_PLOW = 0.02425


def normal_quantile(p) -> np.ndarray:
    p = np.asarray(p, dtype=float)
    if np.any(p <= 0) or np.any(p >= 1):
        raise ValueError("quantile probabilities must lie in (0, 1)")
    out = np.empty_like(p)
    lo, hi = p < _PLOW, p > 1.0 - _PLOW
    mid = ~(lo | hi)
    if np.any(mid):
        q = p[mid] - 0.5
        rr = q * q
        out[mid] = np.polyval(_A, rr) * q / np.polyval(_B, rr)
    for sel, sign, pp in ((lo, 1.0, p), (hi, -1.0, 1.0 - p)):
        if np.any(sel):
            q = np.sqrt(-2.0 * np.log(pp[sel]))
            out[sel] = sign * np.polyval(_C, q) / np.polyval(_D, q)
    return out


@dataclass
class QQData:
    component: str
    q_theory: np.ndarray
    q_empirical: np.ndarray
    correlation: float
    subband: int = -1


def _qq(x: np.ndarray, nq: int, comp: str) -> QQData:
    sd = float(np.std(x))
    if sd == 0.0:
        raise ValueError(f"{comp} part has zero variance")
    z = (x - float(np.mean(x))) / sd
    pos = (np.arange(1, nq + 1) - 0.5) / nq
    qe = np.quantile(z, pos)
    qt = normal_quantile(pos)
    return QQData(comp, qt, qe, float(np.corrcoef(qt, qe)[0, 1]))


def qq_data(residual, n_quantiles: int = 100):
    """Quantile pairs of the real and imaginary parts (src/diagnostics.py:127-149)."""
    res = np.asarray(residual).ravel()
    if n_quantiles < 10:
        raise ValueError(f"need at least 10 quantiles, got {n_quantiles}")
    if res.size < n_quantiles:
        raise ValueError(f"sample of size {res.size} too small for {n_quantiles} quantiles")
    return _qq(res.real, n_quantiles, "real"), _qq(res.imag, n_quantiles, "imag")
