# Round measurements on one B200 (run under gpurun): bench lines, reference arm,
# ncu launch list and full captures (one lane, so every launch covers the whole
# batch as in bench.py's instrumented pass).  TAG names the outputs (e.g. r01e).
set -x
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01e}
python bench.py > gpurun_out/${TAG}_bench_cfg1.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
for c in cfg0 cfg2 cfg3 cfg4_r4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>> gpurun_out/${TAG}_bench.err; echo $c rc=$?
done
VDAMP_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo ncu1 rc=$?
VDAMP_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"synth256|col_pass256|analysis256|sure_select" -s 40 -c 5 -f -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu2 rc=$?
