"""CPU oracle for the VDAMP hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference VDAMP reconstruction
loop (``csmri.vdamp.run`` and everything it calls).  It is the checker that
the CUDA path is compared against; it is NEVER imported by the product
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it.

Parity pin: ``tests/golden/make_golden.py`` runs the reference itself
(``/root/reference/pkg/src/csmri``, importable in the build container only)
on seeded inputs and stores its outputs under ``tests/golden/``;
``tests/test_oracle.py`` checks this restatement against every fixture.

Reference citations use ``src/`` = ``/root/reference/pkg/src/csmri/``.
Everything here is complex128 / float64, like the reference, unless a caller
passes float32 magnitudes to :func:`threshold_scan` (the teacher-forced fp32
check of the GPU path).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SQRT2 = math.sqrt(2.0)
ALPHA_CLAMP = 1.0 - 1e-9          # src/vdamp.py:25
TAU_FLOOR = 1e-300                # src/vdamp.py:118
NMSE_FLOOR_DB = -320.0            # src/diagnostics.py:17
ORIENTS = ("horizontal", "vertical", "diagonal")


# --------------------------------------------------------------------------
# Subband layout (src/wavelet.py:43-63)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Band:
    scale: int
    orientation: str
    offset: int
    length: int
    shape: tuple


def band_table(height: int, width: int, scales: int) -> list[Band]:
    """Flat coefficient layout: approx_s, then (H, V, D) from scale s to 1.

    Follows src/wavelet.py:52-61 (scale-major, coarse first, each block
    row-major).  Raises ValueError like src/wavelet.py:45-51.
    """
    if scales < 1:
        raise ValueError(f"scales must be >= 1, got {scales}")
    if height % (1 << scales) or width % (1 << scales):
        raise ValueError(f"({height}, {width}) not divisible by 2^{scales}")
    bands = []
    hs, ws = height >> scales, width >> scales
    bands.append(Band(scales, "approx", 0, hs * ws, (hs, ws)))
    pos = hs * ws
    for lev in range(scales, 0, -1):
        h, w = height >> lev, width >> lev
        for o in ORIENTS:
            bands.append(Band(lev, o, pos, h * w, (h, w)))
            pos += h * w
    return bands


def band_index(scales: int, level: int, orient: int) -> int:
    """Subband number of detail (level, orient) with orient 0=H, 1=V, 2=D."""
    return 1 + 3 * (scales - level) + orient


# --------------------------------------------------------------------------
# Orthonormal Haar (src/wavelet.py:107-148, 169-181)
# --------------------------------------------------------------------------
def _split(a):
    # one analysis level: axis 0 (rows) first, then axis 1; taps are
    # divided by sqrt(2) exactly as src/wavelet.py:109-114 does.
    lo = (a[0::2] + a[1::2]) / SQRT2
    hi = (a[0::2] - a[1::2]) / SQRT2
    return ((lo[:, 0::2] + lo[:, 1::2]) / SQRT2,   # ll
            (lo[:, 0::2] - lo[:, 1::2]) / SQRT2,   # lh = "horizontal"
            (hi[:, 0::2] + hi[:, 1::2]) / SQRT2,   # hl = "vertical"
            (hi[:, 0::2] - hi[:, 1::2]) / SQRT2)   # hh = "diagonal"


def _merge(ll, lh, hl, hh):
    # inverse of _split (src/wavelet.py:118-129)
    h2, w2 = ll.shape
    lo = np.empty((h2, 2 * w2), dtype=np.result_type(ll, lh))
    hi = np.empty_like(lo)
    lo[:, 0::2] = (ll + lh) / SQRT2
    lo[:, 1::2] = (ll - lh) / SQRT2
    hi[:, 0::2] = (hl + hh) / SQRT2
    hi[:, 1::2] = (hl - hh) / SQRT2
    out = np.empty((2 * h2, 2 * w2), dtype=lo.dtype)
    out[0::2] = (lo + hi) / SQRT2
    out[1::2] = (lo - hi) / SQRT2
    return out


def dwt(image: np.ndarray, scales: int) -> np.ndarray:
    image = np.asarray(image)
    bands = band_table(image.shape[0], image.shape[1], scales)
    out = np.empty(image.size, dtype=np.complex128)
    a = image
    for lev in range(1, scales + 1):
        a, *details = _split(a)
        j0 = band_index(scales, lev, 0)
        for o in range(3):
            b = bands[j0 + o]
            out[b.offset:b.offset + b.length] = details[o].ravel()
    out[:bands[0].length] = a.ravel()
    return out


def idwt(coeffs: np.ndarray, height: int, width: int, scales: int) -> np.ndarray:
    bands = band_table(height, width, scales)

    def blk(j):
        b = bands[j]
        return coeffs[b.offset:b.offset + b.length].reshape(b.shape)

    a = blk(0)
    for lev in range(scales, 0, -1):
        j0 = band_index(scales, lev, 0)
        a = _merge(a, blk(j0), blk(j0 + 1), blk(j0 + 2))
    return a


# --------------------------------------------------------------------------
# Centered unitary FFT and masked operators (src/fourier.py:52-77)
# --------------------------------------------------------------------------
def fft2c(x):
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(x), norm="ortho"))


def ifft2c(k):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(k), norm="ortho"))


def mask_indices(sampled: np.ndarray) -> np.ndarray:
    """Row-major sampled positions (src/fourier.py:26)."""
    return np.flatnonzero(np.asarray(sampled, dtype=bool).ravel())


def forward(x, idx):
    return fft2c(x).ravel()[idx]


def adjoint(y, idx, shape):
    k = np.zeros(shape[0] * shape[1], dtype=np.complex128)
    k[idx] = y
    return ifft2c(k.reshape(shape))


# --------------------------------------------------------------------------
# Subband spectra and tau (src/vdamp.py:41-78)
# --------------------------------------------------------------------------
def haar_profile_1d(n: int, level: int, high: bool) -> np.ndarray:
    """|fft1c(atom)|^2 of the 1D Haar atom at ``level`` on a length-n grid.

    The 2D atom of every subband is separable (row atom x column atom), so
    the reference's 2D profile |fft2c(idwt(unit))|^2 (src/vdamp.py:41-51)
    equals an outer product of two of these.
    """
    atom = np.zeros(n, dtype=np.complex128)
    m = 1 << level
    amp = 2.0 ** (-level / 2.0)
    if high:
        atom[: m // 2] = amp
        atom[m // 2: m] = -amp
    else:
        atom[:m] = amp
    f = np.fft.fftshift(np.fft.fft(np.fft.ifftshift(atom), norm="ortho"))
    return np.abs(f) ** 2


def band_profile_factors(height, width, scales):
    """Per subband (row profile over axis 0, column profile over axis 1)."""
    out = []
    for b in band_table(height, width, scales):
        lev = b.scale
        row_high = b.orientation in ("vertical", "diagonal")     # hl, hh
        col_high = b.orientation in ("horizontal", "diagonal")   # lh, hh
        out.append((haar_profile_1d(height, lev, row_high),
                    haar_profile_1d(width, lev, col_high)))
    return out


def spectra(height, width, scales) -> np.ndarray:
    """(S, H, W) profiles, built separably."""
    return np.stack([np.outer(a, b) for a, b in band_profile_factors(height, width, scales)])


def spectra_from_atoms(height, width, scales) -> np.ndarray:
    """The reference's own construction (src/vdamp.py:41-51): one atom per band."""
    bands = band_table(height, width, scales)
    out = np.empty((len(bands), height, width))
    unit = np.zeros(height * width, dtype=np.complex128)
    for j, b in enumerate(bands):
        unit[b.offset] = 1.0
        out[j] = np.abs(fft2c(idwt(unit, height, width, scales))) ** 2
        unit[b.offset] = 0.0
    return out


def masked_profiles(prof: np.ndarray, idx: np.ndarray) -> np.ndarray:
    return prof.reshape(prof.shape[0], -1)[:, idx]          # src/vdamp.py:54-56


def tau_update(z, idx, probs, noise_var, mprof) -> np.ndarray:
    """tau_j = sum_w m_j(w) p^-1 [(p^-1 - 1)|z|^2 + sigma^2]  (src/vdamp.py:59-78)."""
    if z.shape != (idx.size,):
        raise ValueError("residual length != mask count")
    pinv = 1.0 / probs.ravel()[idx]
    w = pinv * ((pinv - 1.0) * np.abs(z) ** 2 + noise_var)
    return mprof @ w


# --------------------------------------------------------------------------
# SURE threshold selection (src/denoise.py:62-118, 147-178)
# --------------------------------------------------------------------------
def threshold_scan(mag_sorted: np.ndarray, tau: float):
    """Exact SURE argmin over {0} U {|r_i|} U interior stationary points.

    Restates src/denoise.py:62-118.  Candidate t = m_i splits the sorted
    magnitudes at the end of the tie run containing i (entries equal to t
    are zeroed).  Between consecutive candidates the risk is the quadratic
    c t^2 - tau*inv*t + const, whose stationary point tau*inv/(2c) is also a
    candidate when it lies strictly inside the gap.  Sums are float64 even
    when ``mag_sorted`` is float32.  Ties in risk go to the smaller t.
    Returns (t, count_above, sum_inv_above).
    """
    m = np.asarray(mag_sorted, dtype=np.float64)
    n = m.size
    # cumulative squares from below, cumulative inverses from above
    csq = np.zeros(n + 1)
    np.cumsum(m * m, out=csq[1:])
    safe = np.where(m > 0, m, 1.0)
    inv = np.where(m > 0, 1.0 / safe, 0.0)
    cinv = np.zeros(n + 1)
    cinv[:n] = np.cumsum(inv[::-1])[::-1]
    # split index of each candidate (0 first, then each m_i): first index
    # whose magnitude is strictly greater than the candidate value
    cand = np.empty(n + 1)
    cand[0] = 0.0
    cand[1:] = m
    split = np.searchsorted(m, cand, side="right")
    cnt = n - split
    below = csq[split]
    above_inv = cinv[split]
    risk = below + cand ** 2 * cnt - n * tau + tau * (2.0 * cnt - cand * above_inv)
    nxt = np.empty(n + 1)
    nxt[:n] = m
    nxt[n] = np.inf
    with np.errstate(divide="ignore", invalid="ignore"):
        ts = tau * above_inv / (2.0 * cnt)
    inside = (cnt > 0) & (ts > cand) & (ts < nxt)
    risk_s = np.full(n + 1, np.inf)
    risk_s[inside] = (below[inside] + ts[inside] ** 2 * cnt[inside] - n * tau
                      + tau * (2.0 * cnt[inside] - ts[inside] * above_inv[inside]))
    t_all = np.concatenate((cand, np.where(inside, ts, np.inf)))
    r_all = np.concatenate((risk, risk_s))
    best_r = r_all.min()
    tied = np.flatnonzero(r_all == best_r)
    k = tied[np.argmin(t_all[tied])]
    kk = k % (n + 1)
    return float(t_all[k]), float(cnt[kk]), float(above_inv[kk])


def soft(r, t):
    """r * max(1 - t/|r|, 0), boundary |r| == t -> 0 (src/denoise.py:38-45)."""
    mag = np.abs(r)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = np.where(mag > t, 1.0 - t / np.maximum(mag, 1e-300), 0.0)
    return r * g


def sure_risk(r, tau, t):
    """Direct SURE evaluation (src/denoise.py:48-59); a test cross-check."""
    mag = np.abs(r)
    a = mag > t
    return float(np.sum(np.minimum(mag, t) ** 2)) - r.size * tau + tau * float(np.sum(2.0 - t / mag[a]))


def denoise_colored(r, tau, bands):
    """Per-subband SURE soft threshold -> (w_hat, alpha, lambda, t)."""
    if len(tau) != len(bands):
        raise ValueError("tau length != number of subbands")
    if np.any(np.asarray(tau) <= 0):
        raise ValueError("subband noise variances must be > 0")
    out = np.empty_like(r)
    S = len(bands)
    alpha = np.empty(S)
    lam = np.empty(S)
    thr = np.empty(S)
    for j, b in enumerate(bands):
        seg = r[b.offset:b.offset + b.length]
        t, cnt, inv = threshold_scan(np.sort(np.abs(seg)), tau[j])
        out[b.offset:b.offset + b.length] = soft(seg, t)
        alpha[j] = (cnt - 0.5 * t * inv) / b.length
        lam[j] = t / tau[j]
        thr[j] = t
    return out, alpha, lam, thr


# --------------------------------------------------------------------------
# One VDAMP iteration, finalize, full loop (src/vdamp.py:99-197)
# --------------------------------------------------------------------------
@dataclass
class Problem:
    y: np.ndarray            # (n,) complex, aligned with idx
    idx: np.ndarray          # (n,) row-major sampled positions
    probs: np.ndarray        # (H, W) sampling probabilities in (0, 1]
    noise_var: float
    scales: int

    def __post_init__(self):
        self.H, self.W = self.probs.shape
        self.bands = band_table(self.H, self.W, self.scales)
        self.mprof = masked_profiles(spectra(self.H, self.W, self.scales), self.idx)
        self.pinv = 1.0 / self.probs.ravel()[self.idx]


@dataclass
class Step:
    r_tilde_in: np.ndarray
    r: np.ndarray
    z: np.ndarray
    tau: np.ndarray
    thresholds: np.ndarray
    alpha: np.ndarray
    lambdas: np.ndarray
    clamped: bool
    w_hat: np.ndarray
    r_tilde: np.ndarray


def step(p: Problem, r_tilde: np.ndarray) -> Step:
    """Algorithm 1 lines 3-8 (src/vdamp.py:99-144)."""
    shape = (p.H, p.W)
    z = p.y - forward(idwt(r_tilde, p.H, p.W, p.scales), p.idx)
    r = r_tilde + dwt(adjoint(p.pinv * z, p.idx, shape), p.scales)
    tau = tau_update(z, p.idx, p.probs, p.noise_var, p.mprof)
    tau_f = np.maximum(tau, TAU_FLOOR)
    w_hat, alpha, lam, _ = denoise_colored(r, tau_f, p.bands)
    clamped = bool(np.any(alpha >= ALPHA_CLAMP))
    if clamped:
        alpha = np.minimum(alpha, ALPHA_CLAMP)
    nxt = np.empty_like(r)
    for j, b in enumerate(p.bands):
        sl = slice(b.offset, b.offset + b.length)
        nxt[sl] = (w_hat[sl] - alpha[j] * r[sl]) * (1.0 / (1.0 - alpha[j]))
    return Step(r_tilde, r, z, tau, lam * tau, alpha, lam, clamped, w_hat, nxt)


def finalize(w_hat, p: Problem):
    """x = idwt(w); x + adjoint(y - forward(x))  (src/vdamp.py:147-150)."""
    x = idwt(w_hat, p.H, p.W, p.scales)
    return x + adjoint(p.y - forward(x, p.idx), p.idx, (p.H, p.W))


def nmse_db(x_hat, x0):
    """src/diagnostics.py:21-34."""
    ref = float(np.vdot(x0, x0).real)
    if ref == 0.0:
        raise ValueError("reference signal is identically zero")
    e = x_hat - x0
    num = float(np.vdot(e, e).real)
    if num == 0.0:
        return NMSE_FLOOR_DB
    return max(10.0 * math.log10(num / ref), NMSE_FLOOR_DB)


def subband_nmse(r, w0, bands):
    """src/diagnostics.py:37-51 (NaN for zero-energy subbands)."""
    out = np.empty(len(bands))
    for j, b in enumerate(bands):
        sl = slice(b.offset, b.offset + b.length)
        ref = float(np.vdot(w0[sl], w0[sl]).real)
        if ref == 0.0:
            out[j] = float("nan")
            continue
        e = r[sl] - w0[sl]
        num = float(np.vdot(e, e).real)
        out[j] = max(10.0 * math.log10(num / ref), NMSE_FLOOR_DB) if num else NMSE_FLOOR_DB
    return out


@dataclass
class Record:
    k: int
    tau: np.ndarray
    thresholds: np.ndarray
    lambdas: np.ndarray
    alphas: np.ndarray
    alpha_clamped: bool
    nmse_db: float | None = None
    subband_nmse_db: np.ndarray | None = None


@dataclass
class Result:
    x_hat: np.ndarray
    records: list = field(default_factory=list)
    snapshots: dict = field(default_factory=dict)
    steps: list = field(default_factory=list)


def _round_c64(v):
    return v.astype(np.complex64).astype(np.complex128)


def run(y, idx, probs, noise_var, scales, n_iters, ground_truth=None,
        keep_r_iters=(), keep_steps=False, c64_state=False) -> Result:
    """The reconstruction loop (src/vdamp.py:153-197).

    ``c64_state=True`` is the complex64 floor of SURVEY A.3 (not a reference
    mode): the iteration state r~_{k+1} and w_hat_k are rounded to complex64
    after every iteration, everything else stays float64.  The distance of
    this run from the plain run is the deviation that storing the state in
    complex64 alone causes; the fp32 CUDA path is judged against it."""
    if n_iters < 1:
        raise ValueError(f"need at least one iteration, got {n_iters}")
    p = Problem(np.asarray(y, dtype=np.complex128), np.asarray(idx), np.asarray(probs, float),
                float(noise_var), scales)
    w0 = dwt(ground_truth, scales) if ground_truth is not None else None
    res = Result(None)
    rt = np.zeros(p.H * p.W, dtype=np.complex128)
    st = None
    for k in range(n_iters):
        st = step(p, rt)
        if c64_state:
            st.r_tilde = _round_c64(st.r_tilde)
            st.w_hat = _round_c64(st.w_hat)
        rec = Record(k, st.tau.copy(), st.thresholds.copy(), st.lambdas.copy(),
                     st.alpha.copy(), st.clamped)
        if ground_truth is not None:
            rec.nmse_db = nmse_db(finalize(st.w_hat, p), ground_truth)
            rec.subband_nmse_db = subband_nmse(st.r, w0, p.bands)
        if k in keep_r_iters:
            res.snapshots[k] = st.r.copy()
        if keep_steps:
            res.steps.append(st)
        res.records.append(rec)
        rt = st.r_tilde
    res.x_hat = finalize(st.w_hat, p)
    return res


# --------------------------------------------------------------------------
# Baselines on the same operators (src/baselines.py) -- SURVEY §8f row 3
# --------------------------------------------------------------------------
SURE_IT_TAU_FLOOR = 1e-30         # src/baselines.py:23


def gradient_step(r_tilde, y, idx, shape, scales):
    """r~ + Psi F^H M^T (y - M F Psi^H r~), unit step (src/baselines.py:41-43)."""
    resid = y - forward(idwt(r_tilde, shape[0], shape[1], scales), idx)
    return r_tilde + dwt(adjoint(resid, idx, shape), scales)


def _momentum(t_m):
    t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t_m * t_m))
    return t_next, (t_m - 1.0) / t_next


def fista(y, idx, shape, lam, n_iters, scales=4, ground_truth=None):
    """Accelerated soft thresholding, one global threshold (src/baselines.py:54-91).
    Returns (x_hat, nmse_curve or None)."""
    if lam <= 0:
        raise ValueError("lam must be > 0")
    if n_iters < 1:
        raise ValueError("need at least one iteration")
    w_hat = np.zeros(shape[0] * shape[1], dtype=np.complex128)
    rt = w_hat
    t_m = 1.0
    nm = []
    for _ in range(n_iters):
        g = gradient_step(rt, y, idx, shape, scales)
        w_new = soft(g, lam)
        t_m, beta = _momentum(t_m)
        rt = w_new + beta * (w_new - w_hat)
        w_hat = w_new
        if ground_truth is not None:
            nm.append(nmse_db(idwt(w_hat, shape[0], shape[1], scales), ground_truth))
    return idwt(w_hat, shape[0], shape[1], scales), (nm if ground_truth is not None else None)


def sure_it(y, idx, shape, w0, n_iters, scales=4, ground_truth=None):
    """SURE-tuned thresholding with the oracle scalar error level (src/baselines.py:115-164).
    Returns (x_hat, taus, thresholds, nmse_curve or None)."""
    bands = band_table(shape[0], shape[1], scales)
    N = shape[0] * shape[1]
    w_hat = np.zeros(N, dtype=np.complex128)
    rt = w_hat
    t_m = 1.0
    taus, thr, nm = [], [], []
    for _ in range(n_iters):
        r = gradient_step(rt, y, idx, shape, scales)
        e = r - w0
        tau_k = max(float(np.vdot(e, e).real) / N, SURE_IT_TAU_FLOOR)
        tau = np.full(len(bands), tau_k)
        w_new, _, lam, _ = denoise_colored(r, tau, bands)
        t_m, beta = _momentum(t_m)
        rt = w_new + beta * (w_new - w_hat)
        w_hat = w_new
        taus.append(tau)
        thr.append(lam * tau)
        if ground_truth is not None:
            nm.append(nmse_db(idwt(w_hat, shape[0], shape[1], scales), ground_truth))
    return (idwt(w_hat, shape[0], shape[1], scales), np.array(taus), np.array(thr),
            nm if ground_truth is not None else None)


def tune_lambda(y, idx, shape, x0, budget_iters, grid, scales=4):
    """Smallest-NMSE threshold on a grid, ties keep the smaller (src/baselines.py:94-112)."""
    grid = np.sort(np.asarray(grid, dtype=float))
    if grid.size == 0:
        raise ValueError("empty lambda grid")
    best, best_nm = None, np.inf
    for lam in grid:
        x, _ = fista(y, idx, shape, float(lam), budget_iters, scales)
        s = nmse_db(x, x0)
        if s < best_nm:
            best, best_nm = float(lam), s
    return best
