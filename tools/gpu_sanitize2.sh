cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -q -m gpu -x -k "attention or ragged or sequence_parallel or merge" -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/attn_bench.py 8 24 4608 128
timeout 120 python tools/attn_bench.py 8 24 4429 64
for w in tiny flux_block; do
  for t in memcheck racecheck synccheck; do
    echo "=== $t $w"
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py $w > gpurun_out/san_${t}_${w}.log 2>&1
    echo "rc=$?"; tail -3 gpurun_out/san_${t}_${w}.log
  done
done
