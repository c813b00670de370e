cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), json.dumps({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()}))'; }
A="--warmup 3 --no-cpu-baseline --no-extras --no-e2e"
for i in 1 2; do
echo "cfg1 nostream: $(VDAMP_LIB=$PWD/build/nostream.so run $A --steps 20)"
echo "cfg1 stream:   $(run $A --steps 20)"
done
echo "cfg4 nostream: $(VDAMP_LIB=$PWD/build/nostream.so run $A --steps 5 --config cfg4_r4)"
echo "cfg4 stream:   $(run $A --steps 5 --config cfg4_r4)"
echo "cfg0 nostream: $(VDAMP_LIB=$PWD/build/nostream.so run $A --steps 5 --config cfg0)"
echo "cfg0 stream:   $(run $A --steps 5 --config cfg0)"
