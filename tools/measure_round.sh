set -x
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_r01c_ref.json 2> gpurun_out/bench_r01c_ref.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r01c.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sure_select -s 40 -c 1 -f -o gpurun_out/prof_r01c_select python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_r01c.log 2>&1; echo ncu2 rc=$?
