set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/r2b_pytest.log 2>&1
tail -25 gpurun_out/r2b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
tail -3 gpurun_out/r2b_smoke.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
cat gpurun_out/r2b_bench.json
timeout 300 python tools/attn_bench.py > gpurun_out/r2b_attn.log 2>&1
tail -20 gpurun_out/r2b_attn.log
