cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), json.dumps({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()}))'; }
timeout 600 python -m pytest tests/test_gpu_workloads.py -x -q -k "nmse_beside or parseval or lanes" 2>&1 | tail -3
A="--config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e"
echo "cfg2 default: $(run $A)"
echo "cfg2 forced cluster: $(VDAMP_CLUSTER=1 run $A)"
echo "cfg2 b16 default: $(run $A --batch 16)"
echo "cfg2 b16 forced cluster: $(VDAMP_CLUSTER=1 run $A --batch 16)"
CFG=cfg2 bash tools/s5_ncu_cfg.sh 2>/dev/null | head -14
