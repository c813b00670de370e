cd $GRAFT_REPO_ROOT
VDAMP_GRAPHS=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for G in 1 0; do
  VDAMP_GRAPHS=$G python bench.py --no-cpu-baseline > gpurun_out/g.json 2>gpurun_out/g.err
  python -c "import json; d=json.load(open('gpurun_out/g.json')); print('graphs $G', round(d['value']), round(d['e2e']['value']), round(d['e2e'].get('sync_call_value')), d['gpu_launches'])" || tail -3 gpurun_out/g.err
done; done
