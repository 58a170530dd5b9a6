cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sd3.py tests/test_gpu_parity.py tests/test_gpu_zz_attn_split.py -q -x > gpurun_out/d64_tests.log 2>&1; tail -1 gpurun_out/d64_tests.log
for r in 1 2; do
  timeout 120 python tools/attn_bench.py 8 24 4608 64 2>&1 | tail -1
  timeout 120 python tools/attn_bench.py 8 24 4429 64 2>&1 | tail -1
  timeout 120 python tools/attn_bench.py 2>&1 | tail -1
done
timeout 400 python bench.py --workload sd3m --no-cpu-baseline > gpurun_out/d64_sd3m.json 2>/dev/null; python tools/bench_brief.py gpurun_out/d64_sd3m.json | head -2
