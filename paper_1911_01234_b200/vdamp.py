"""VDAMP reconstruction loop on B200 -- drop-in for ``csmri.vdamp`` (src/vdamp.py).

``run(y, mask, pmap, noise_var, scales, n_iters, ground_truth=None,
keep_r_iters=())`` keeps the reference signature, return types and errors.
The whole loop (K1..K4 per iteration, finalize) runs on the device through
``libvdamp_b200.so``; the host only validates, uploads and reads back.

Extensions (keyword-only): ``precision`` ("fp64" = the reference's
complex128 arithmetic, the parity mode and the default; "fp32" = complex64
throughput mode) and ``device``.  ``run_batch`` reconstructs many
independent images in one launch sequence.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .denoise import SubbandVector
from .fourier import SamplingMask
from .trace import IterationRecord, RunTrace
from .wavelet import SubbandLayout, WaveletCoeffs

ALPHA_CLAMP = 1.0 - 1e-9          # src/vdamp.py:25
NMSE_FLOOR_DB = -320.0            # src/diagnostics.py:17


def _probs(pmap, shape):
    probs = np.asarray(getattr(pmap, "probs", pmap), dtype=np.float64)
    if probs.shape != tuple(shape):
        raise ValueError(f"probability map shape {probs.shape} != mask shape {tuple(shape)}")
    if np.any(probs <= 0) or np.any(probs > 1):
        raise ValueError("probabilities must lie in (0, 1]")
    return probs


def _nmse_db(err: float, ref: float) -> float:
    # src/diagnostics.py:21-34
    if ref == 0.0:
        raise ValueError("reference signal is identically zero")
    if err == 0.0:
        return NMSE_FLOOR_DB
    return max(10.0 * np.log10(err / ref), NMSE_FLOOR_DB)


def _subband_nmse(err: np.ndarray, ref: np.ndarray) -> np.ndarray:
    # src/diagnostics.py:37-51 (NaN sentinel for zero-energy subbands)
    out = np.full(err.shape, np.nan)
    nz = ref != 0.0
    with np.errstate(divide="ignore"):
        v = np.where(err > 0, 10.0 * np.log10(np.where(err > 0, err, 1.0) / np.where(nz, ref, 1.0)), NMSE_FLOOR_DB)
    out[nz] = np.maximum(v[nz], NMSE_FLOOR_DB)
    return out


@dataclass
class BatchInputs:
    """Host-side concatenation of a batch's measurements (what the C ABI takes)."""

    y: np.ndarray
    indices: np.ndarray
    counts: np.ndarray
    probs: np.ndarray
    shared_probs: bool
    noise_var: np.ndarray
    height: int
    width: int


def prepare_batch(ys, masks, pmaps, noise_vars) -> BatchInputs:
    """Validate like the reference (src/fourier.py:62-77, src/sampling.py:45-46) and concatenate."""
    masks = list(masks)
    B = len(masks)
    if B < 1:
        raise ValueError("empty batch")
    ys = list(ys)
    if len(ys) != B:
        raise ValueError("one measurement vector per mask required")
    shape = masks[0].shape
    for m in masks:
        if m.shape != shape:
            raise ValueError("all images of a batch must share one shape")
    if not isinstance(pmaps, (list, tuple)):
        probs = _probs(pmaps, shape)
        shared = True
    else:
        if len(pmaps) != B:
            raise ValueError("one probability map per mask required")
        if all(p is pmaps[0] for p in pmaps):
            probs, shared = _probs(pmaps[0], shape), True
        else:
            probs, shared = np.stack([_probs(p, shape) for p in pmaps]), False
    nv = np.asarray(noise_vars, dtype=np.float64).reshape(-1)
    if nv.size == 1 and B > 1:
        nv = np.full(B, float(nv[0]))
    if nv.shape != (B,):
        raise ValueError("one noise variance per image required")
    if np.any(nv < 0):
        raise ValueError("noise variance must be >= 0")
    for y, m in zip(ys, masks):
        if np.shape(y) != (m.n,):
            raise ValueError(f"measurement length {np.shape(y)} != mask count {m.n}")
    counts = np.array([m.n for m in masks], dtype=np.int64)
    idx = np.concatenate([m.indices for m in masks]).astype(np.int64)
    y = np.concatenate([np.asarray(v) for v in ys])
    return BatchInputs(y, idx, counts, probs, shared, nv, shape[0], shape[1])


def _records(trace_np, nmse_np, b, n_iters, wall):
    recs = []
    for k in range(n_iters):
        tr = trace_np[k, b]
        tau = tr[:, 0].copy()
        lam = tr[:, 2].copy()
        rec = IterationRecord(
            k=k, wall_time=float(wall[k]) if np.ndim(wall) else float(wall), tau=tau, thresholds=lam * tau,
            lambdas=lam,
            alphas=tr[:, 3].copy(), alpha_clamped=bool(np.any(tr[:, 5] != 0)))
        if nmse_np is not None:
            rec.nmse_db = _nmse_db(float(nmse_np[k, b, 0]), float(nmse_np[k, b, 1]))
            rec.subband_nmse_db = _subband_nmse(tr[:, 6], tr[:, 7])
        recs.append(rec)
    return recs


def run_batch(ys, masks, pmaps, noise_vars, scales, n_iters, ground_truths=None, keep_r_iters=(),
              *, precision="fp64", device=None, return_tensor=False, keep_device=False):
    """VDAMP on a batch of independent images (one launch sequence for all).

    Returns (x_hat (B, H, W) complex ndarray, [RunTrace per image]).  With
    ``keep_device`` the r snapshots stay on the device: ``traces[0].device_snapshots[k]``
    is the (B, N) tensor of r_k (no per-image host copies).
    """
    import torch
    from .plan import get_plan
    if n_iters < 1:
        raise ValueError(f"need at least one iteration, got {n_iters}")
    masks = list(masks)
    inp = prepare_batch(ys, masks, pmaps, noise_vars)
    layout = SubbandLayout.create(inp.height, inp.width, scales)
    B = len(masks)
    t0 = time.perf_counter()
    plan = get_plan(inp.height, inp.width, scales, B, precision, device)
    plan.set_measurements(inp.y, inp.indices, inp.counts, inp.probs, inp.noise_var, inp.shared_probs)
    gt = None
    if ground_truths is not None:
        gt = np.stack([np.asarray(g) for g in ground_truths])
        if gt.shape != (B, inp.height, inp.width):
            raise ValueError("ground truth shape mismatch")
        plan.set_ground_truth(gt)
    else:
        plan.set_ground_truth(None)
    torch.cuda.synchronize(plan.device)
    precompute = time.perf_counter() - t0
    trace = plan.new_trace(n_iters)
    nmse = (torch.zeros((n_iters, B, _lib.NMSE_FIELDS), dtype=torch.float64, device=plan.device)
            if gt is not None else None)
    snaps = {k: plan.empty_coeffs() for k in keep_r_iters if 0 <= k < n_iters} or None
    plan.set_iteration_timing(True)
    x = plan.run(n_iters, trace=trace, nmse=nmse, snapshots=snaps)
    ms, images = plan.iteration_times(n_iters)
    plan.set_iteration_timing(False)
    # each iteration's own device time (src/vdamp.py:176-179), per image of its stream
    wall = ms / 1e3 / max(images, 1)
    trace_np = trace.cpu().numpy()
    nmse_np = nmse.cpu().numpy() if nmse is not None else None
    traces = []
    for b in range(B):
        rt = RunTrace("vdamp", _records(trace_np, nmse_np, b, n_iters, wall), precompute)
        if snaps and not keep_device:
            for k, t in snaps.items():
                rt.r_snapshots[k] = WaveletCoeffs(t[b].cpu().numpy().astype(np.complex128), layout)
        traces.append(rt)
    if keep_device and traces:
        traces[0].device_snapshots = snaps or {}
    if return_tensor:
        return x, traces
    return x.cpu().numpy().astype(np.complex128), traces


def run(y, mask: SamplingMask, pmap, noise_var, scales, n_iters, ground_truth=None, keep_r_iters=(),
        *, precision="fp64", device=None):
    """Full reconstruction loop (src/vdamp.py:153-197); trace metrics only with ground truth."""
    if n_iters < 1:
        raise ValueError(f"need at least one iteration, got {n_iters}")
    SubbandLayout.create(mask.shape[0], mask.shape[1], scales)
    x, traces = run_batch([y], [mask], pmap, [noise_var], scales, n_iters,
                          None if ground_truth is None else [ground_truth], keep_r_iters,
                          precision=precision, device=device)
    return x[0], traces[0]


# ---------------------------------------------------------------------------
# Step-wise interface (src/vdamp.py:81-150)
# ---------------------------------------------------------------------------
@dataclass
class VdampState:
    r_tilde: WaveletCoeffs
    r: WaveletCoeffs | None = None
    z: np.ndarray | None = None          # fused on device, not materialised
    tau: SubbandVector | None = None
    w_hat: WaveletCoeffs | None = None
    alpha: SubbandVector | None = None
    thresholds: np.ndarray | None = None
    lambdas: SubbandVector | None = None
    k: int = 0
    alpha_clamped: bool = False


def initial_state(layout: SubbandLayout) -> VdampState:
    return VdampState(WaveletCoeffs(np.zeros(layout.size, dtype=np.complex128), layout))


def iterate(state: VdampState, y, mask: SamplingMask, pmap, noise_var, spectra=None,
            masked_profiles=None, *, precision="fp64", device=None) -> VdampState:
    """One iteration from state.r_tilde (src/vdamp.py:99-144); spectra args are accepted and unused
    (the plan builds the separable subband spectra on the device)."""
    import torch
    from .plan import get_plan
    lay = state.r_tilde.layout
    inp = prepare_batch([y], [mask], pmap, [noise_var])
    plan = get_plan(lay.image_height, lay.image_width, lay.scales, 1, precision, device)
    plan.set_measurements(inp.y, inp.indices, inp.counts, inp.probs, inp.noise_var, inp.shared_probs)
    plan.set_ground_truth(None)
    rt = plan.to_device(state.r_tilde.values, plan.cdtype).reshape(1, -1).contiguous()
    r = plan.empty_coeffs()
    rn = plan.empty_coeffs()
    wh = plan.empty_coeffs()
    tr = torch.zeros((1, plan.S, _lib.TRACE_FIELDS), dtype=torch.float64, device=plan.device)
    plan.iterate(rt, r, rn, wh, tr)
    t = tr[0].cpu().numpy()
    tau = t[:, 0].copy()
    lam = t[:, 2].copy()
    as_np = lambda v: v[0].cpu().numpy().astype(np.complex128)
    return VdampState(
        r_tilde=WaveletCoeffs(as_np(rn), lay), r=WaveletCoeffs(as_np(r), lay), z=None,
        tau=SubbandVector(tau, "variance"), w_hat=WaveletCoeffs(as_np(wh), lay),
        alpha=SubbandVector(t[:, 3].copy(), "derivative"), thresholds=lam * tau,
        lambdas=SubbandVector(lam, "weight"), k=state.k + 1,
        alpha_clamped=bool(np.any(t[:, 5] != 0)))


def finalize(w_hat: WaveletCoeffs, y, mask: SamplingMask, *, precision="fp64", device=None) -> np.ndarray:
    """Exact data consistency: replace sampled frequencies by y (src/vdamp.py:147-150)."""
    from .plan import get_plan
    lay = w_hat.layout
    inp = prepare_batch([y], [mask], np.ones(mask.shape), [0.0])
    plan = get_plan(lay.image_height, lay.image_width, lay.scales, 1, precision, device)
    plan.set_measurements(inp.y, inp.indices, inp.counts, inp.probs, inp.noise_var, True)
    w = plan.to_device(w_hat.values, plan.cdtype).reshape(1, -1).contiguous()
    out = plan.empty_images()
    plan.finalize(w, out)
    return out[0].cpu().numpy().astype(np.complex128)


# ---------------------------------------------------------------------------
# Repeated batched reconstruction (serving / benchmark entry point)
# ---------------------------------------------------------------------------
class BatchReconstructor:
    """Reconstruct batches of B images of one geometry, reusing the device plan.

    ``__call__`` takes the concatenated measurements (see :func:`prepare_batch`)
    as numpy arrays or torch tensors -- host (ideally pinned) or device -- and
    returns x_hat (B, H, W).  With ``out`` a pinned host tensor the result is
    copied back asynchronously into it; the call synchronises before returning.
    """

    def __init__(self, height, width, scales, batch, *, precision="fp32", device=None):
        from .plan import get_plan
        SubbandLayout.create(height, width, scales)
        self.plan = get_plan(height, width, scales, batch, precision, device)
        self._x = self.plan.empty_images()

    def upload(self, inp: BatchInputs, pin=True):
        """Host BatchInputs -> torch host tensors (pinned) ready for __call__."""
        import torch
        t = lambda a, dt: (torch.from_numpy(np.ascontiguousarray(a)).to(dt).pin_memory() if pin
                           else torch.from_numpy(np.ascontiguousarray(a)).to(dt))
        return dict(y=t(inp.y, self.plan.cdtype), indices=t(inp.indices, torch.int64),
                    counts=inp.counts, probs=t(inp.probs, torch.float64), noise_var=inp.noise_var,
                    shared_probs=inp.shared_probs)

    def __call__(self, y, indices, counts, probs, noise_var, n_iters, *, shared_probs=True, out=None,
                 stream=None, sync=True):
        if n_iters < 1:
            raise ValueError(f"need at least one iteration, got {n_iters}")
        p = self.plan
        p.set_measurements(y, indices, counts, probs, noise_var, shared_probs, stream=stream,
                           sync_validation=False)
        x = p.run(n_iters, x_hat=self._x, stream=stream)
        if out is not None:
            out.copy_(x, non_blocking=True)
            x = out
        if sync:
            import torch
            torch.cuda.current_stream(p.device).synchronize() if stream is None else stream.synchronize()
            p.measurement_status(wait=True)
        return x


class StreamingReconstructor:
    """Pipelined batches: host->device copies of batch k+1 and the device->host
    copy of batch k-1 overlap the reconstruction of batch k.  With ``depth`` > 1
    the reconstructions of ``depth`` consecutive batches also run side by side on
    their own plans and compute streams; measured slower on cfg1 (64 x 256^2:
    depth 1 / 2 / 3 = 503k / 408k / 317k img-iter/s: a batch's image lanes already
    fill the GPU), so the default is one reconstruction at a time.

    ``submit`` takes pinned host tensors (see :meth:`BatchReconstructor.upload`)
    and a pinned host ``out`` tensor (B, H, W); it returns at once.  ``wait``
    blocks until every submitted batch has landed in its ``out``.  Inputs of a
    submitted batch must not be modified until its copy has finished
    (``depth`` + 1 batches in flight at most; ``submit`` blocks beyond that).
    Results are bitwise those of :class:`BatchReconstructor` at any depth.
    """

    def __init__(self, height, width, scales, batch, *, precision="fp32", device=None, depth=1):
        import torch
        from .plan import Plan, get_plan
        SubbandLayout.create(height, width, scales)
        if depth < 1:
            raise ValueError(f"depth must be >= 1, got {depth}")
        self.plan = get_plan(height, width, scales, batch, precision, device)
        dev = self.plan.device
        # one plan (workspace) and compute stream per batch in flight on the device
        self.plans = [self.plan] + [Plan(height, width, scales, batch, precision, dev.index)
                                    for _ in range(depth - 1)]
        self.computes = [torch.cuda.Stream(dev) for _ in range(depth)]
        self.compute = self.computes[0]
        self.copy = torch.cuda.Stream(dev)          # host -> device
        self.copy_out = torch.cuda.Stream(dev)      # device -> host (never queued behind an upload)
        self.depth = depth
        ns = depth + 1                              # staged inputs / x_hat slots
        self._x = [self.plan.empty_images() for _ in range(ns)]
        self._stage = [None] * ns
        self._ev_out = [None] * ns          # D2H of slot finished
        self._k = 0

    upload = BatchReconstructor.upload

    def submit(self, host, n_iters, out):
        import torch
        if n_iters < 1:
            raise ValueError(f"need at least one iteration, got {n_iters}")
        s = self._k % (self.depth + 1)
        p, compute = self.plans[self._k % self.depth], self.computes[self._k % self.depth]
        self._k += 1
        if self._ev_out[s] is not None:
            self._ev_out[s].synchronize()      # slot s (stage and x) free again
        with torch.cuda.stream(self.copy):
            st = dict(y=host["y"].to(p.device, non_blocking=True),
                      indices=host["indices"].to(p.device, non_blocking=True),
                      probs=host["probs"].to(p.device, non_blocking=True))
            ev_in = torch.cuda.Event()
            ev_in.record(self.copy)
        self._stage[s] = st
        compute.wait_event(ev_in)
        with torch.cuda.stream(compute):
            p.set_measurements(st["y"], st["indices"], host["counts"], st["probs"], host["noise_var"],
                               host.get("shared_probs", True), stream=compute, sync_validation=False)
            p.run(n_iters, x_hat=self._x[s], stream=compute)
            ev_done = torch.cuda.Event()
            ev_done.record(compute)
        self.copy_out.wait_event(ev_done)
        with torch.cuda.stream(self.copy_out):
            out.copy_(self._x[s], non_blocking=True)
            ev_out = torch.cuda.Event()
            ev_out.record(self.copy_out)
        self._ev_out[s] = ev_out
        return out

    def wait(self):
        """Block until every submitted batch has landed; raises ValueError if the
        device flagged the measurements of any of them."""
        for e in self._ev_out:
            if e is not None:
                e.synchronize()
        for p in self.plans:
            p.measurement_status(wait=True)
