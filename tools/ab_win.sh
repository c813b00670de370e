# A/B of sure_win32 (VDAMP_PRUNE=1) against the full sort (=0): SURE parity tests, bench values, launch list
cd $GRAFT_REPO_ROOT
VDAMP_PRUNE=1 python -m pytest tests/test_gpu_parity.py -x -q -k "sure_select or denoise" 2>&1 | tail -2
VDAMP_PRUNE=0 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 10 --quick 2>&1 | grep "value\|sure_select"
for cfgs in "256 1" "256 0" "512 1" "128 1"; do set -- $cfgs
  echo "WIN4=$1 WINSIDE=$2"
  VDAMP_WIN4=$1 VDAMP_WINSIDE=$2 VDAMP_PRUNE=1 python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 10 --quick 2>&1 | grep "value\|sure_select"
done
VDAMP_PRUNE=1 VDAMP_LANES=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file /tmp/wl.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > /tmp/wl.log 2>&1
python tools/profile_summary.py /tmp/wl.csv /tmp/win | grep "sure_"
