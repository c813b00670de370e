cd $GRAFT_REPO_ROOT
for f in 0 1; do
VDAMP_F256=$f timeout 600 ncu --set full --import-source on --clock-control none -k regex:col_pass -s 12 -c 1 -f -o gpurun_out/col_f$f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_col_f$f.log 2>&1; echo ncu$f rc=$?
done
