import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VDAMP_LIB"] = os.path.join(ROOT, "paper_1911_01234_b200", "libvdamp_b200_phase.so")
import numpy as np
from paper_1911_01234_b200 import _lib, vdamp, workload
w = workload.make_workload("cfg2", batch=32)
x, tr = vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 5, 45, keep_r_iters=(44,), precision="fp32")
lib = _lib.load()
buf = (ctypes.c_longlong * (64 * 64 * 4))()
lib.vdamp_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.check(lib.vdamp_debug_phase_times(buf, 64))
a = np.frombuffer(buf, dtype=np.int64).reshape(64, 64, 4)[:32, :16, :3].sum(-1)
idx = np.dstack(np.unravel_index(np.argsort(-a.ravel())[:6], a.shape))[0]
for b, j in idx:
    r = tr[b].r_snapshots[44].subband(j)
    m = np.abs(r.astype(np.complex64)).astype(np.float32)
    u, c = np.unique(m, return_counts=True)
    print(f"img {b} band {j} cycles {a[b, j]} n {m.size} min {m.min():.3g} max {m.max():.3g} zeros {(m == 0).sum()} distinct {u.size} maxdup {c.max()} nonfinite {(~np.isfinite(m)).sum()}")
