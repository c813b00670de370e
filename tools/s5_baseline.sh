# session-5 baseline: gpu tests, bench, lanes x graphs sweep, ncu source capture of sure_win32
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5_gputest.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s5_gputest.log
python bench.py --no-extras > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo bench rc=$?
for cfg in "4 0" "4 1" "6 1" "8 1" "8 0" "2 1"; do
  set -- $cfg
  echo "lanes=$1 graphs=$2: $(VDAMP_LANES=$1 VDAMP_GRAPHS=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-extras 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')"
done
TAG=s5win
VDAMP_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sure_win32" -s 20 -c 2 -f -o /tmp/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_source.csv 2>/dev/null; echo src rc=$?
python tools/ncu_lines.py /tmp/${TAG}_source.csv "sure_win32<(int)512" 3000 > gpurun_out/${TAG}_lines512.txt 2>&1
python tools/ncu_lines.py /tmp/${TAG}_source.csv "sure_win32<(int)256" 3000 > gpurun_out/${TAG}_lines256.txt 2>&1
head -5 gpurun_out/${TAG}_lines512.txt
