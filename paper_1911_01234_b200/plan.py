"""Device plan: workspace, uploads and launches for one image geometry.

A :class:`Plan` owns the C-side ``vdamp_plan_t`` for (H, W, scales, batch,
precision, device).  Torch provides the device memory of inputs/outputs and
the stream; all compute is in libvdamp_b200.so.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

PRECISIONS = {"fp32": _lib.FP32, "fp64": _lib.FP64}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1911_01234_b200 needs a CUDA device (B200); no CPU fallback")
    return torch


@dataclass(frozen=True)
class PlanKey:
    height: int
    width: int
    scales: int
    batch: int
    precision: str
    device: int


class Plan:
    def __init__(self, height, width, scales, batch=1, precision="fp64", device=None):
        torch = _torch()
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")
        if device is None:
            device = torch.cuda.current_device()
        self.key = PlanKey(int(height), int(width), int(scales), int(batch), precision, int(device))
        self.H, self.W, self.scales, self.B = int(height), int(width), int(scales), int(batch)
        self.N = self.H * self.W
        self.precision = precision
        self.device = torch.device("cuda", int(device))
        self.cdtype = torch.complex64 if precision == "fp32" else torch.complex128
        self.rdtype = torch.float32 if precision == "fp32" else torch.float64
        lib = _lib.load()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.vdamp_plan_create(self.H, self.W, self.scales, self.B,
                                             PRECISIONS[precision], int(device), ctypes.byref(h)))
        self._h = h
        self.S = 1 + 3 * self.scales
        off = (ctypes.c_int64 * self.S)()
        ln = (ctypes.c_int64 * self.S)()
        _lib.check(lib.vdamp_plan_layout(self._h, off, ln))
        self.offsets = np.array(off[:], dtype=np.int64)
        self.lengths = np.array(ln[:], dtype=np.int64)
        self.has_measurements = False

    # ------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.load().vdamp_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if not self._h:
            raise RuntimeError("plan is closed")
        return self._h

    def workspace_bytes(self) -> int:
        v = ctypes.c_size_t()
        _lib.check(_lib.load().vdamp_plan_workspace_bytes(self.handle, ctypes.byref(v)))
        return int(v.value)

    # ------------------------------------------------------------------
    def empty_images(self):
        torch = _torch()
        return torch.empty((self.B, self.H, self.W), dtype=self.cdtype, device=self.device)

    def empty_coeffs(self):
        torch = _torch()
        return torch.empty((self.B, self.N), dtype=self.cdtype, device=self.device)

    def to_device(self, a, dtype):
        """numpy / torch (pinned or not) -> contiguous device tensor of dtype."""
        torch = _torch()
        if isinstance(a, torch.Tensor):
            t = a
        else:
            t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=self.device, dtype=dtype, non_blocking=True).contiguous()

    def set_measurements(self, y, indices, counts, probs, noise_var, shared_probs=False, stream=None,
                         sync_validation=True):
        """y: concatenated (sum n_b,) complex; indices int64 same length;
        counts (B,); probs (B,H,W) or (H,W) when shared_probs; noise_var (B,).

        The device checks every index (range, repeats) and the probability at it;
        a flagged batch raises ValueError here (``sync_validation``) or, on the
        pipelined path (``sync_validation=False``), from the first later call that
        finds the check landed, or from :meth:`measurement_status`."""
        torch = _torch()
        if sync_validation != getattr(self, "_sync_val", True):
            _lib.check(_lib.load().vdamp_set_validation(self.handle, int(bool(sync_validation))))
        self._sync_val = bool(sync_validation)
        y_d = self.to_device(y, self.cdtype)
        i_d = self.to_device(indices, torch.int64)
        p_d = self.to_device(probs, torch.float64)
        cnt = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
        nv = np.ascontiguousarray(np.asarray(noise_var, dtype=np.float64))
        if cnt.shape != (self.B,) or nv.shape != (self.B,):
            raise ValueError("counts and noise_var need one entry per image")
        if y_d.numel() != int(cnt.sum()) or i_d.numel() != int(cnt.sum()):
            raise ValueError("y / indices length does not match the mask counts")
        stride = 0 if shared_probs else self.N
        if p_d.numel() != (self.N if shared_probs else self.B * self.N):
            raise ValueError("probability map has the wrong size")
        _lib.check(_lib.load().vdamp_set_measurements(
            self.handle, _lib.ptr(y_d), _lib.ptr(i_d),
            cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _lib.ptr(p_d), stride,
            nv.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _lib.stream_ptr(stream)))
        self._keep = (y_d, i_d, p_d)
        self.has_measurements = True

    def measurement_status(self, wait=True):
        """Raise ValueError if any measurements set so far were flagged by the device check."""
        _lib.check(_lib.load().vdamp_measurement_status(self.handle, int(bool(wait))))

    def set_ground_truth(self, x0, stream=None):
        if x0 is None:
            _lib.check(_lib.load().vdamp_set_ground_truth(self.handle, None, _lib.stream_ptr(stream)))
            return
        x_d = self.to_device(x0, self.cdtype).reshape(self.B, self.H, self.W).contiguous()
        _lib.check(_lib.load().vdamp_set_ground_truth(self.handle, _lib.ptr(x_d), _lib.stream_ptr(stream)))

    def run(self, n_iters, x_hat=None, trace=None, nmse=None, snapshots=None, stream=None):
        if x_hat is None:
            x_hat = self.empty_images()
        snaps = None
        if snapshots is not None:
            arr = (ctypes.c_void_p * n_iters)()
            for k in range(n_iters):
                arr[k] = snapshots[k].data_ptr() if snapshots.get(k) is not None else None
            snaps = ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))
        _lib.check(_lib.load().vdamp_run(self.handle, int(n_iters), _lib.ptr(x_hat), _lib.ptr(trace),
                                         _lib.ptr(nmse), snaps, _lib.stream_ptr(stream)))
        return x_hat

    def new_trace(self, n_iters):
        torch = _torch()
        return torch.zeros((n_iters, self.B, self.S, _lib.TRACE_FIELDS), dtype=torch.float64,
                           device=self.device)

    def iterate(self, r_tilde, r=None, r_tilde_next=None, w_hat=None, trace=None, stream=None):
        _lib.check(_lib.load().vdamp_iterate(self.handle, _lib.ptr(r_tilde), _lib.ptr(r),
                                             _lib.ptr(r_tilde_next), _lib.ptr(w_hat), _lib.ptr(trace),
                                             _lib.stream_ptr(stream)))

    def dwt(self, image, coeffs, stream=None):
        _lib.check(_lib.load().vdamp_dwt(self.handle, _lib.ptr(image), _lib.ptr(coeffs), _lib.stream_ptr(stream)))

    def idwt(self, coeffs, image, stream=None):
        _lib.check(_lib.load().vdamp_idwt(self.handle, _lib.ptr(coeffs), _lib.ptr(image), _lib.stream_ptr(stream)))

    def fft2c(self, x, out, inverse=False, stream=None):
        _lib.check(_lib.load().vdamp_fft2c(self.handle, _lib.ptr(x), _lib.ptr(out), int(bool(inverse)),
                                           _lib.stream_ptr(stream)))

    def finalize(self, w_hat, x_hat, stream=None):
        _lib.check(_lib.load().vdamp_finalize(self.handle, _lib.ptr(w_hat), _lib.ptr(x_hat),
                                              _lib.stream_ptr(stream)))

    def denoise_colored(self, r, tau, w_hat=None, trace=None, stream=None):
        _lib.check(_lib.load().vdamp_denoise_colored(self.handle, _lib.ptr(r), _lib.ptr(tau), _lib.ptr(w_hat),
                                                     _lib.ptr(trace), _lib.stream_ptr(stream)))

    # instrumentation
    def set_timing(self, enable: bool):
        _lib.check(_lib.load().vdamp_set_timing(self.handle, int(bool(enable))))

    def kernel_times(self):
        ms = (ctypes.c_double * _lib.KERNEL_CLASSES)()
        n = (ctypes.c_int64 * _lib.KERNEL_CLASSES)()
        _lib.check(_lib.load().vdamp_kernel_times(self.handle, ms, n))
        return {name: (float(ms[i]), int(n[i])) for i, name in enumerate(_lib.KERNEL_CLASS_NAMES)}

    def set_graphs(self, enable: bool):
        _lib.check(_lib.load().vdamp_set_graphs(self.handle, int(bool(enable))))

    def set_lanes(self, lanes: int):
        """Run the batch as `lanes` image ranges on their own streams (0 = default).  With the
        default iteration-major launch order the trace, NMSE records and snapshots ride on
        the lanes too (each lane writes its image range)."""
        _lib.check(_lib.load().vdamp_set_lanes(self.handle, int(lanes)))

    def set_iteration_timing(self, enable: bool):
        _lib.check(_lib.load().vdamp_set_iteration_timing(self.handle, int(bool(enable))))

    def iteration_times(self, n_iters):
        """(ms per iteration, images sharing each timed stream) of the last vdamp_run."""
        ms = (ctypes.c_double * n_iters)()
        im = ctypes.c_int()
        _lib.check(_lib.load().vdamp_iteration_times(self.handle, int(n_iters), ms, ctypes.byref(im)))
        return np.array(ms[:], dtype=np.float64), int(im.value)

    def launch_count(self, reset=False) -> int:
        v = ctypes.c_int64()
        _lib.check(_lib.load().vdamp_launch_count(self.handle, ctypes.byref(v), int(bool(reset))))
        return int(v.value)


_CACHE: dict = {}


def get_plan(height, width, scales, batch=1, precision="fp64", device=None) -> Plan:
    """Cached plan per geometry (workspace reuse across calls)."""
    torch = _torch()
    if device is None:
        device = torch.cuda.current_device()
    key = PlanKey(int(height), int(width), int(scales), int(batch), precision, int(device))
    p = _CACHE.get(key)
    if p is None or not p._h:
        p = Plan(height, width, scales, batch, precision, device)
        _CACHE[key] = p
    return p


def clear_plans():
    for p in _CACHE.values():
        p.close()
    _CACHE.clear()
