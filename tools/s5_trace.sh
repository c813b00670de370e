cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
A="--steps 10 --warmup 3 --no-cpu-baseline --no-extras --no-e2e --with-trace"
echo "cfg1 trace overlap=0: $(VDAMP_NMSE_OVERLAP=0 run $A)"
echo "cfg1 trace overlap=1: $(run $A)"
echo "cfg1 trace overlap=1 graphs=0: $(VDAMP_GRAPHS=0 run $A)"
echo "cfg4 trace overlap=0: $(VDAMP_NMSE_OVERLAP=0 run --config cfg4_r4 $A)"
echo "cfg4 trace overlap=1: $(run --config cfg4_r4 $A)"
echo "cfg0 trace overlap=0: $(VDAMP_NMSE_OVERLAP=0 run --config cfg0 $A)"
echo "cfg0 trace overlap=1: $(run --config cfg0 $A)"
echo "cfg1 fp64 trace overlap=0: $(VDAMP_NMSE_OVERLAP=0 run --precision fp64 $A)"
echo "cfg1 fp64 trace overlap=1: $(run --precision fp64 $A)"
