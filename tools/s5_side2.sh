cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
A="--warmup 3 --no-cpu-baseline --no-extras --no-e2e"
for i in 1 2; do
echo "cfg1 side2=0: $(run $A --steps 20)"
echo "cfg1 side2=1: $(VDAMP_SIDE2=1 run $A --steps 20)"
done
echo "cfg4 side2=0: $(run $A --steps 5 --config cfg4_r4)"
echo "cfg4 side2=1: $(VDAMP_SIDE2=1 run $A --steps 5 --config cfg4_r4)"
echo "cfg2 side2=0: $(run $A --steps 5 --config cfg2)"
echo "cfg2 side2=1: $(VDAMP_SIDE2=1 run $A --steps 5 --config cfg2)"
echo "cfg1 b16 side2=0: $(run $A --steps 10 --batch 16)"
echo "cfg1 b16 side2=1: $(VDAMP_SIDE2=1 run $A --steps 10 --batch 16)"
