# shared-memory carve-out preference A/B (session 5)
cd $GRAFT_REPO_ROOT
run() { python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d.get("e2e") or {}; print(round(d["value"]), round(e.get("value",0)), round(e.get("depth1_value",0)))'; }
export VDAMP_GRAPHS=1
for c in -1 100 75 50; do
  echo "cfg1 carveout=$c: $(VDAMP_CARVEOUT=$c run --steps 20 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
for l in 6 8; do
  echo "cfg1 carveout=100 lanes=$l: $(VDAMP_CARVEOUT=100 VDAMP_LANES=$l run --steps 20 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
echo "cfg1 carveout=100 e2e depth 2: $(VDAMP_CARVEOUT=100 run --steps 20 --warmup 3 --no-cpu-baseline --no-extras --e2e-depth 2)"
for c in -1 100; do
  echo "cfg2 carveout=$c: $(VDAMP_GRAPHS=0 VDAMP_CARVEOUT=$c run --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
  echo "cfg4 carveout=$c: $(VDAMP_GRAPHS=0 VDAMP_CARVEOUT=$c run --config cfg4_r4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
