# ncu --set full of one iteration's kernels (synth, col, analysis, both SURE kernels), cfg1 bench workload
cd $GRAFT_REPO_ROOT
TAG=${TAG:-cur}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"synth|col_pass|analysis|sure_select" -s 40 -c 5 -f -o gpurun_out/iter_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_iter_$TAG.log 2>&1; echo ncu rc=$?
