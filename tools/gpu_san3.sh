cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 120 python tools/attn_bench.py 8 24 4608 128; done
git_stash_note="(o_done per item)"
for w in tiny flux_block; do
  t=racecheck; echo "=== $t $w"
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py $w > gpurun_out/san_${t}_${w}.log 2>&1
  echo "rc=$?"; tail -2 gpurun_out/san_${t}_${w}.log
done
