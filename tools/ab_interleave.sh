cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for I in 1 0; do
  VDAMP_INTERLEAVE=$I python bench.py --no-cpu-baseline > gpurun_out/il.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/il.json')); print('interleave $I', round(d['value']), round(d['e2e']['value']), d['e2e'].get('sync_call_value'))"
done; done
