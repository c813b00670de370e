cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]))'; }
A="--warmup 3 --no-cpu-baseline --no-extras --no-e2e"
for c in 0 4 8 16 32 0 8; do
echo "cfg1 winfull_ctas=$c: $(VDAMP_WINFULL_CTAS=$c run $A --steps 20)"
done
echo "cfg1 winfull off (timing only): $(VDAMP_WINFULL=0 run $A --steps 20)"
for c in 0 8; do
echo "cfg4 winfull_ctas=$c: $(VDAMP_WINFULL_CTAS=$c run $A --steps 5 --config cfg4_r4)"
echo "cfg2 winfull_ctas=$c: $(VDAMP_WINFULL_CTAS=$c run $A --steps 5 --config cfg2)"
done
