# Bitwise A/B of the in-tree library against build/prev.so (e.g. a build of the previous commit):
# GPU tests on the in-tree build, then cfg1 / cfg2 reconstructions compared bit for bit.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for spec in "cfg1 8 30" "cfg2 2 10"; do
  set -- $spec
  VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so python tools/cmp_run.py /tmp/a_$1.npz $1 $2 $3
  VDAMP_LIB=$PWD/build/prev.so python tools/cmp_run.py /tmp/b_$1.npz $1 $2 $3
  python -c "
import numpy as np
A=np.load('/tmp/a_$1.npz'); B=np.load('/tmp/b_$1.npz')
for k in A.files: print('$1', k, 'bitwise' if np.array_equal(A[k],B[k]) else 'DIFF %g' % np.nanmax(np.abs(A[k]-B[k])))
"
done
