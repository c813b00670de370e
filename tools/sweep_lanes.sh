# bench value vs image lanes (and a repeat for the run-to-run spread)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for l in 1 2 3 4 6 8; do
  echo -n "rep $rep lanes $l: "; VDAMP_LANES=$l python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 10 --quick 2>&1 | grep "value" | cut -c1-40
done; done
