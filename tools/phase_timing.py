"""Per-phase clocks of sure_select (debug build): python tools/phase_timing.py"""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VDAMP_LIB"] = os.path.join(ROOT, "paper_1911_01234_b200", "libvdamp_b200_phase.so")
import numpy as np
from paper_1911_01234_b200 import _lib, vdamp, workload
w = workload.make_workload("cfg1", batch=64)
vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 4, 3, precision="fp32")
buf = (ctypes.c_longlong * (64 * 64 * 4))()
lib = _lib.load()
lib.vdamp_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_phase_times(buf, 64))
a = np.frombuffer(buf, dtype=np.int64).reshape(64, 64, 4)[:, :13, :3]
lens = [256] * 4 + [1024] * 3 + [4096] * 3 + [16384] * 3
for j in range(13):
    m = a[:, j, :].mean(0)
    print(f"subband {j:2d} n={lens[j]:5d}  load+sort {m[0]:9.0f}  scan {m[1]:9.0f}  argmin {m[2]:7.0f} cycles")

buf2 = (ctypes.c_longlong * (64 * 64 * 6))()
lib.vdamp_debug_csort_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_csort_times(buf2, 64))
c = np.frombuffer(buf2, dtype=np.int64).reshape(64, 64, 6)[:, 10:13, :5].mean((0, 1))
print("counting sort (n=16384) cycles: minmax %.0f  hist %.0f  scan %.0f  scatter %.0f  fixup %.0f" % tuple(c))
