# cluster SURE selection (sure_winc): tests, then cfg0 / cfg3 A/B (session 5)
cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), json.dumps({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()}))'; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -5
echo "cfg0 cluster=0: $(VDAMP_CLUSTER=0 run --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg0 cluster=1: $(run --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg3 cluster=0: $(VDAMP_CLUSTER=0 run --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg3 cluster16=0: $(VDAMP_CLUSTER16=0 run --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg3 cluster16=1: $(run --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
echo "cfg1 batch=4: $(run --config cfg1 --batch 4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
CFG=cfg3 bash tools/s5_ncu_cfg.sh | head -16
