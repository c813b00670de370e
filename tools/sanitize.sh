# compute-sanitizer over tools/sanitize_case.py (run under gpurun); summaries -> gpurun_out/
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
for tool in memcheck synccheck racecheck initcheck; do
  for case in 256 64 512 sure1024; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $case \
      > gpurun_out/${TAG}_sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_sanitize_${tool}_${case}.log | tail -1)"
  done
done
