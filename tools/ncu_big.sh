# ncu of the large-subband SURE kernels on cfg2 (16 slices)
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"big_|sure_select" -c 5 -f -o gpurun_out/big python bench.py --config cfg2 --batch 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_big.log 2>&1; echo rc=$?
