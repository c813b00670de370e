cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), json.dumps({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()}))'; }
A="--warmup 3 --no-cpu-baseline --no-extras --no-e2e"
echo "cfg1: $(run $A --steps 20)"
echo "cfg1: $(run $A --steps 20)"
echo "cfg1 old lib: $(VDAMP_LIB=$PWD/build/nostream.so run $A --steps 20)"
echo "cfg4: $(run $A --steps 5 --config cfg4_r4)"
echo "cfg2: $(run $A --steps 5 --config cfg2)"
echo "cfg0: $(run $A --steps 5 --config cfg0)"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
