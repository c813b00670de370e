"""Per-phase clocks of sure_select (debug build): python tools/phase_timing.py"""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VDAMP_LIB"] = os.path.join(ROOT, "paper_1911_01234_b200", "libvdamp_b200_phase.so")
import numpy as np
from paper_1911_01234_b200 import _lib, vdamp, workload
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
w = workload.make_workload(cfg, batch=nb)
NIT = int(sys.argv[3]) if len(sys.argv) > 3 else 3
vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, w.config.scales, NIT, precision=os.environ.get("PREC", "fp32"))
buf = (ctypes.c_longlong * (64 * 64 * 4))()
lib = _lib.load()
lib.vdamp_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_phase_times(buf, 64))
S = 1 + 3 * w.config.scales
a = np.frombuffer(buf, dtype=np.int64).reshape(64, 64, 4)[:nb, :S, :3]
from paper_1911_01234_b200.wavelet import SubbandLayout
lens = [b.length for b in SubbandLayout.create(w.config.size, w.config.size, w.config.scales).subbands]
for j in range(S):
    m = a[:, j, :].mean(0)
    print(f"subband {j:2d} n={lens[j]:6d}  load+sort {m[0]:9.0f}  scan {m[1]:9.0f}  argmin {m[2]:7.0f} cycles")

buf2 = (ctypes.c_longlong * (64 * 64 * 8))()
lib.vdamp_debug_csort_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_csort_times(buf2, 64))
c6 = np.frombuffer(buf2, dtype=np.int64).reshape(64, 64, 8)[:nb, S - 3:S, :]
print("TMA landed after %.0f cycles, keys built after %.0f (16384-key subbands)" % (c6[..., 5].mean(), c6[..., 6].mean()))
c = c6[..., :5].mean((0, 1))
print("counting sort (n=16384) cycles: minmax+coarse %.0f  table+fine hist %.0f  check+scan %.0f  scatter %.0f  bucket sort %.0f" % tuple(c))

buf3 = (ctypes.c_longlong * (64 * 64 * 5))()
lib.vdamp_debug_scan_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_scan_times(buf3, 64))
c3 = np.frombuffer(buf3, dtype=np.int64).reshape(64, 64, 5)[:nb, :S, :]
for j in range(S):
    m = c3[:, j, :].mean(0)
    print(f"scan subband {j:2d}: pass1 {m[0]:7.0f}  block scans {m[1]:7.0f}  keys {m[2]:7.0f}  barrier {m[3]:7.0f}  merge {m[4]:7.0f}")

buf4 = (ctypes.c_longlong * (64 * 64 * 10))()
if hasattr(lib, "vdamp_debug_prune_times"):
    lib.vdamp_debug_prune_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
    _lib.check(lib.vdamp_debug_prune_times(buf4, 64))
    c4 = np.frombuffer(buf4, dtype=np.int64).reshape(64, 64, 10)[:nb, :S, :]
    for j in range(S):
        if lens[j] < 4096:
            continue
        m = c4[:, j, :].mean(0)
        ok = (c4[:, j, 8] == 1).mean()
        print(f"prune subband {j:2d} n={lens[j]}: hist {m[0]:6.0f} coarse {m[1]:6.0f} pass1 {m[2]:6.0f} "
              f"fine {m[3]:6.0f} pass2 {m[4]:6.0f} sort {m[5]:6.0f} scan {m[6]:6.0f} | span {m[6-0]*0:.0f}"
              f"list {m[7]:7.1f} (max {c4[:, j, 7].max()}) pruned {ok:.2f}")
