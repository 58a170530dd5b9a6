cd $GRAFT_REPO_ROOT
for w in tiny flux_block; do
  for t in memcheck racecheck synccheck; do
    echo "=== $t $w"
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py $w > gpurun_out/san_${t}_${w}.log 2>&1
    echo "rc=$?"; tail -4 gpurun_out/san_${t}_${w}.log
  done
done
