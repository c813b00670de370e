cd $GRAFT_REPO_ROOT
VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so python tools/cmp_run.py /tmp/a.npz cfg1 8 30
VDAMP_LIB=$PWD/build/prev.so python tools/cmp_run.py /tmp/b.npz cfg1 8 30
VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so python tools/cmp_run.py /tmp/a2.npz cfg2 2 10
VDAMP_LIB=$PWD/build/prev.so python tools/cmp_run.py /tmp/b2.npz cfg2 2 10
python -c "
import numpy as np
for a,b in (('a','b'),('a2','b2')):
    A=np.load('/tmp/'+a+'.npz'); B=np.load('/tmp/'+b+'.npz')
    for k in A.files: print(a, k, 'bitwise' if np.array_equal(A[k],B[k]) else 'DIFF %g' % np.nanmax(np.abs(A[k]-B[k])))
"
bash tools/ab_bench.sh; bash tools/ab_bench.sh
