# Session-5 measurement set (run under gpurun): GPU tests, default bench (all configs), reference
# arm, ncu launch list (one lane, direct launches, so each launch covers the whole batch as in
# bench.py's instrumented pass) and one --set full capture of the per-iteration kernels.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02s5}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_gputest.log
python bench.py > gpurun_out/${TAG}_bench_cfg1_with_configs.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
VDAMP_GRAPHS=0 VDAMP_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu1 rc=$?
VDAMP_GRAPHS=0 VDAMP_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"synth256|col_pass256|analysis256|sure_select|sure_win32" -s 40 -c 6 -f -o /tmp/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu2 rc=$?
python tools/ncu_stalls.py /tmp/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_full_summary.txt 2>&1
VDAMP_GRAPHS=0 timeout 600 ncu --set full --clock-control none -k regex:"sure_winc" -s 12 -c 2 -f -o /tmp/${TAG}_winc python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu_winc.log 2>&1; echo ncu3 rc=$?
python tools/ncu_stalls.py /tmp/${TAG}_winc.ncu-rep > gpurun_out/${TAG}_ncu_winc_summary.txt 2>&1
ls -la gpurun_out/${TAG}*
