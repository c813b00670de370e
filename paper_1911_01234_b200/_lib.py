"""ctypes binding of the C ABI in include/vdamp_b200.h.

The shared library ``libvdamp_b200.so`` is built in-tree by
``__graft_entry__.build()`` (or ``make -C paper_1911_01234_b200/csrc``).
There is no fallback: if the library or a CUDA device is missing, every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os

# The image lanes and their side streams (up to 8 compute streams plus the copy streams of the
# streaming API) should each get their own hardware work queue; the CUDA default of 8 lets two
# of them share one, which serialises their kernels.  Read by the CUDA driver at context
# creation, so it only takes effect when this package is imported before CUDA is initialised.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VDAMP_LIB") or os.path.join(_HERE, "libvdamp_b200.so")

VDAMP_OK = 0
VDAMP_ERR_ARG = 1
VDAMP_ERR_SHAPE = 2
VDAMP_ERR_UNSUPPORTED = 3
VDAMP_ERR_CUDA = 4
VDAMP_ERR_OOM = 5
VDAMP_ERR_STATE = 6
FP32 = 0
FP64 = 1
TRACE_FIELDS = 8
NMSE_FIELDS = 2
KERNEL_CLASSES = 6
KERNEL_CLASS_NAMES = ("synth_rowfft", "col_residual", "rowifft_analysis", "sure_select",
                      "finalize", "other")

# every symbol declared in include/vdamp_b200.h: name -> (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "vdamp_last_error": (ctypes.c_char_p, []),
    "vdamp_abi_version": (_I, []),
    "vdamp_plan_create": (_I, [_I, _I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "vdamp_plan_destroy": (_I, [_P]),
    "vdamp_plan_layout": (_I, [_P, _I64P, _I64P]),
    "vdamp_plan_workspace_bytes": (_I, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "vdamp_set_measurements": (_I, [_P, _P, _P, _I64P, _P, ctypes.c_int64, _DP, _P]),
    "vdamp_set_ground_truth": (_I, [_P, _P, _P]),
    "vdamp_run": (_I, [_P, _I, _P, _P, _P, ctypes.POINTER(_P), _P]),
    "vdamp_iterate": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "vdamp_dwt": (_I, [_P, _P, _P, _P]),
    "vdamp_idwt": (_I, [_P, _P, _P, _P]),
    "vdamp_fft2c": (_I, [_P, _P, _P, _I, _P]),
    "vdamp_finalize": (_I, [_P, _P, _P, _P]),
    "vdamp_denoise_colored": (_I, [_P, _P, _P, _P, _P, _P]),
    "vdamp_set_timing": (_I, [_P, _I]),
    "vdamp_kernel_times": (_I, [_P, _DP, _I64P]),
    "vdamp_set_graphs": (_I, [_P, _I]),
    "vdamp_set_lanes": (_I, [_P, _I]),
    "vdamp_mc_accumulate": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "vdamp_baseline_run": (_I, [_P, _I, _I, _P, _P, _P, _P, _P]),
    "vdamp_launch_count": (_I, [_P, _I64P, _I]),
    "vdamp_set_validation": (_I, [_P, _I]),
    "vdamp_measurement_status": (_I, [_P, _I]),
    "vdamp_check_measurements": (_I, [_I, _I, _I, _I64P, _I64P, _DP, ctypes.c_int64, _DP]),
    "vdamp_set_iteration_timing": (_I, [_P, _I]),
    "vdamp_iteration_times": (_I, [_P, _I, _DP, ctypes.POINTER(_I)]),
}

_lib = None


class DimensionError(ValueError):
    """Image dimensions incompatible with the decomposition depth (src/wavelet.py:21-22)."""


def load():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == VDAMP_OK:
        return
    msg = load().vdamp_last_error().decode(errors="replace")
    if rc == VDAMP_ERR_SHAPE:
        raise DimensionError(msg)
    if rc in (VDAMP_ERR_ARG, VDAMP_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == VDAMP_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(f"vdamp error {rc}: {msg}")


def ptr(t) -> ctypes.c_void_p:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return ctypes.c_void_p(None)
    return ctypes.c_void_p(t.data_ptr())


def dptr(t):
    if t is None:
        return ctypes.cast(ctypes.c_void_p(None), _DP)
    return ctypes.cast(ctypes.c_void_p(t.data_ptr()), _DP)


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
