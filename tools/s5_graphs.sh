# graphs on/off across configs; e2e depth sweep (session 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { python bench.py "$@" 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d.get("e2e") or {}; print(round(d["value"]), round(e.get("value",0)), round(e.get("depth1_value",0)), round(e.get("sync_call_value",0)))'; }
timeout 600 python -m pytest tests/test_gpu_workloads.py -x -q -k "streaming or validation or lanes or graph" 2>&1 | tail -3
for g in 0 1; do
  echo "cfg1 graphs=$g (value e2e depth1 sync): $(VDAMP_GRAPHS=$g run --steps 20 --warmup 3 --no-cpu-baseline --no-extras)"
done
for d in 1 2 3; do
  echo "cfg1 graphs=1 e2e-depth=$d: $(VDAMP_GRAPHS=1 run --steps 20 --warmup 3 --no-cpu-baseline --no-extras --e2e-depth $d)"
done
for c in cfg2 cfg3 cfg0 cfg4_r4; do for g in 0 1; do
  echo "$c graphs=$g: $(VDAMP_GRAPHS=$g run --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done; done
for g in 0 1; do
  echo "cfg1 fp64 graphs=$g: $(VDAMP_GRAPHS=$g run --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
  echo "cfg1 trace graphs=$g: $(VDAMP_GRAPHS=$g run --with-trace --steps 10 --warmup 3 --no-cpu-baseline --no-extras --no-e2e)"
done
python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("cfg3 kernels", json.dumps(d["kernels"]))'
python bench.py --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("cfg0 kernels", json.dumps(d["kernels"]))'
