# ncu --set full of the big SURE kernel (one lane, cfg1); per-line summary + rep into gpurun_out/ (TAG env)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-sure}
VDAMP_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sure_select" -s 20 -c 2 -f -o /tmp/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_source.csv 2>/dev/null; echo src rc=$?
python tools/ncu_lines.py /tmp/${TAG}_source.csv "sure_select<float, (int)1024>" 3000 > gpurun_out/${TAG}_lines.txt 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null; echo det rc=$?
ls -la /tmp/${TAG}.ncu-rep
gzip -c /tmp/${TAG}.ncu-rep > gpurun_out/${TAG}.ncu-rep.gz
