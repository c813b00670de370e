cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so python tools/cmp_run.py gpurun_out/new.npz cfg1 8 30
VDAMP_LIB=$PWD/build/prev.so python tools/cmp_run.py gpurun_out/prev.npz cfg1 8 30
VDAMP_LIB=$PWD/paper_1911_01234_b200/libvdamp_b200.so python tools/cmp_run.py gpurun_out/new2.npz cfg2 2 10
VDAMP_LIB=$PWD/build/prev.so python tools/cmp_run.py gpurun_out/prev2.npz cfg2 2 10
python -c "
import numpy as np
for a,b in (('new','prev'),('new2','prev2')):
    A=np.load('gpurun_out/'+a+'.npz'); B=np.load('gpurun_out/'+b+'.npz')
    for k in A.files: print(a, k, 'bitwise' if np.array_equal(A[k],B[k]) else 'DIFF %g' % np.nanmax(np.abs(A[k]-B[k])))
"
bash tools/ab_bench.sh; bash tools/ab_bench.sh
timeout 300 python tools/phase_timing.py 2>&1 | grep -E "scan subband ( [0-9]|1[0-2])"
