# Round-2 profile set (run under gpurun): ncu launch list (one lane, so each launch covers
# the whole batch as in bench.py's instrumented pass) and one --set full capture of the
# four per-iteration kernels; summaries into gpurun_out/ (the .ncu-rep stays on the box,
# a gzip copy is brought back).  TAG names the outputs.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
VDAMP_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu1 rc=$?
VDAMP_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"synth256|col_pass256|analysis256|sure_select|sure_win32" -s 40 -c 5 -f -o /tmp/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu2 rc=$?
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > /tmp/${TAG}_raw.csv 2>/dev/null
python tools/ncu_stalls.py /tmp/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_summary.txt 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_ncu_full_details.csv 2>/dev/null
gzip -c /tmp/${TAG}_full.ncu-rep > gpurun_out/${TAG}_full.ncu-rep.gz
ls -la gpurun_out/${TAG}*
