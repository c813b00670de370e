cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d.get("e2e") or {}; print(round(d["value"]), round(e.get("value",0)))'; }
A="--warmup 3 --no-cpu-baseline --no-extras"
echo "cfg1 default: $(run $A --steps 20)"
for l in 2 3 5 6 8; do
echo "cfg1 lanes=$l: $(VDAMP_LANES=$l run $A --steps 20 --no-e2e)"
done
echo "cfg1 WIN4=128: $(VDAMP_WIN4=128 run $A --steps 20 --no-e2e)"
echo "cfg1 WINFEW=1: $(VDAMP_WINFEW=1 run $A --steps 20 --no-e2e)"
echo "cfg1 trace: $(run $A --steps 10 --no-e2e --with-trace)"
echo "cfg1 fp64: $(run $A --steps 5 --no-e2e --precision fp64)"
echo "cfg0: $(run $A --steps 5 --no-e2e --config cfg0)"
echo "cfg3: $(run $A --steps 5 --no-e2e --config cfg3)"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
