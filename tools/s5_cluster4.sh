cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
echo "cfg0: $(run --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg3: $(run --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
for b in 6 8 12 16 24; do
echo "cfg1 batch=$b default: $(run --config cfg1 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)  forced cluster: $(VDAMP_CLUSTER=1 run --config cfg1 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)  off: $(VDAMP_CLUSTER=0 run --config cfg1 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
for b in 3 4 8; do
echo "cfg2 batch=$b default: $(run --config cfg2 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)  forced cluster: $(VDAMP_CLUSTER=1 run --config cfg2 --batch $b --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
