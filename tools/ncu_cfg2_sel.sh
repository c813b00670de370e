# ncu --set full of the big SURE kernel on cfg2 (16 slices; subbands of 65,536 keys on the single-CTA path)
cd $GRAFT_REPO_ROOT
VDAMP_LANES=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sure_select -s 2 -c 1 -f -o gpurun_out/cfg2sel python bench.py --config cfg2 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg2sel.log 2>&1; echo rc=$?
