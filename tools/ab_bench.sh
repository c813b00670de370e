# A/B: bench value + per-class ms for the in-tree library and build/*.so variants
cd $GRAFT_REPO_ROOT
for lib in paper_1911_01234_b200/libvdamp_b200.so $(ls build/*.so 2>/dev/null); do
  VDAMP_LIB=$PWD/$lib python bench.py --no-cpu-baseline --no-e2e $AB_ARGS > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab.json'))
k=d['kernels']; print('$lib', round(d['value']), {n: round(v['ms_per_step'],3) for n,v in k.items()})"
done
