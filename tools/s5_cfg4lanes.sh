cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
A="--warmup 3 --no-cpu-baseline --no-extras --no-e2e"
for l in 1 2 4; do
echo "cfg4 lanes=$l: $(VDAMP_LANES=$l run $A --steps 5 --config cfg4_r4)"
echo "cfg2 lanes=$l: $(VDAMP_LANES=$l run $A --steps 5 --config cfg2)"
done
echo "cfg2 lanes=3: $(VDAMP_LANES=3 run $A --steps 5 --config cfg2)"
for b in 128 256; do for l in 1 2 4; do
echo "cfg1 batch=$b lanes=$l: $(VDAMP_LANES=$l run $A --steps 5 --batch $b)"
done; done
