cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san3
for spec in "memcheck b16" "racecheck b16" "synccheck b16" "memcheck flux_block" "synccheck flux_block"; do
  set -- $spec
  echo "=== $1 $2"
  timeout 900 compute-sanitizer --tool $1 --print-limit 20 python tools/sanitize_step.py $2 > gpurun_out/san3/${1}_${2}.log 2>&1
  echo "rc=$?"; tail -3 gpurun_out/san3/${1}_${2}.log
done
