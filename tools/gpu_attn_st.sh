cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/att_full.log 2>&1; tail -1 gpurun_out/att_full.log
for r in 1 2; do
  timeout 120 python tools/attn_bench.py 2>&1 | tail -1
  timeout 120 python tools/attn_bench.py 8 24 4429 64 2>&1 | tail -1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/att_cfg3.json 2>/dev/null; python tools/bench_brief.py gpurun_out/att_cfg3.json 2>/dev/null | head -2
