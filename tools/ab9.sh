cd $GRAFT_REPO_ROOT
AB_ARGS="--config cfg2 --steps 5 --warmup 3" bash tools/ab_bench.sh
AB_ARGS="--config cfg3 --steps 3 --warmup 3" bash tools/ab_bench.sh
for L in 2 3 4 5 6 8; do
  VDAMP_LANES=$L python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lanes.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lanes.json')); print('lanes $L', round(d['value']))"
done
