cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
A="--steps 20 --warmup 3 --no-cpu-baseline --no-extras --no-e2e"
echo "default: $(run $A)"
echo "WINFEW=1: $(VDAMP_WINFEW=1 run $A)"
echo "WIN4=128: $(VDAMP_WIN4=128 run $A)"
echo "WIN4=512: $(VDAMP_WIN4=512 run $A)"
echo "WINSIDE=0: $(VDAMP_WINSIDE=0 run $A)"
echo "lanes=3: $(VDAMP_LANES=3 run $A)"
echo "lanes=5: $(VDAMP_LANES=5 run $A)"
echo "interleave=0: $(VDAMP_INTERLEAVE=0 run $A)"
echo "default again: $(run $A)"
