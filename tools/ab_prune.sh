# A/B of the bound-pruned SURE path (VDAMP_PRUNE=1, default) against the full sort (=0):
# thresholds and x_hat of fixed runs, and bench values.  Run under gpurun.
cd $GRAFT_REPO_ROOT
for c in cfg1 cfg4_r8 cfg4_r16 cfg0; do
  VDAMP_PRUNE=0 python tools/cmp_run.py /tmp/p0_$c.npz $c 8 30 2>&1 | tail -1
  VDAMP_PRUNE=1 python tools/cmp_run.py /tmp/p1_$c.npz $c 8 30 2>&1 | tail -1
  python - <<PY
import numpy as np
a = np.load('/tmp/p0_$c.npz'); b = np.load('/tmp/p1_$c.npz')
for k in a.files:
    x, y = a[k], b[k]
    if k.endswith('_thr'):
        d = np.abs(x - y) / np.maximum(np.abs(x), 1e-300)
        print('$c', k, 'thresholds identical', np.mean(x == y), 'max rel diff', d.max(), 'n>1e-9', int((d > 1e-9).sum()), 'of', d.size)
    else:
        print('$c', k, 'x_hat bitwise', np.array_equal(x, y), 'rel', np.linalg.norm(x - y) / np.linalg.norm(x))
PY
done
for v in 0 1; do VDAMP_PRUNE=$v python bench.py --no-extras --no-cpu-baseline --steps 10 --quick; done
