cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), json.dumps({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()}))'; }
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "cfg0: $(run --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg3: $(run --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg1 batch=4: $(run --config cfg1 --batch 4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg1 batch=8: $(run --config cfg1 --batch 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg2 batch=1 cluster=0: $(VDAMP_CLUSTER=0 run --config cfg2 --batch 1 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg2 batch=1 cluster=1: $(run --config cfg2 --batch 1 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg2 batch=2 cluster=0: $(VDAMP_CLUSTER=0 run --config cfg2 --batch 2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg2 batch=2 cluster=1: $(run --config cfg2 --batch 2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
