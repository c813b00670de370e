# large-subband pruning A/B (cfg2 / cfg3, both precisions)
cd $GRAFT_REPO_ROOT
for c in cfg2 cfg3; do for prec in fp32 fp64; do for v in 0 $( [ $prec = fp64 ] && echo 3 || echo 2 ); do
  echo "== $c $prec VDAMP_PRUNE=$v"; VDAMP_PRUNE=$v timeout 600 python bench.py --config $c --precision $prec --no-extras --no-cpu-baseline --no-e2e --steps 3 --quick 2>&1 | grep -E "value|sure|rror"
done; done; done
VDAMP_PRUNE=0 python tools/cmp_run.py /tmp/l0.npz cfg2 4 12; VDAMP_PRUNE=3 python tools/cmp_run.py /tmp/l1.npz cfg2 4 12
python -c "
import numpy as np
a=np.load('/tmp/l0.npz'); b=np.load('/tmp/l1.npz')
for k in a.files:
    x,y=a[k],b[k]
    if k.endswith('_thr'): d=np.abs(x-y)/np.maximum(np.abs(x),1e-300); print(k,'identical',np.mean(x==y),'max rel',d.max())
    else: print(k,'rel',np.linalg.norm(x-y)/np.linalg.norm(x))
"
