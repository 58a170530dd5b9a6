set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $O/nvsmi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 300 python tools/attn_bench.py > $O/attn128.txt 2>&1
timeout 300 python tools/attn_bench.py 8 24 4608 64 > $O/attn64.txt 2>&1
timeout 300 python tools/attn_fa4.py > $O/fa4.txt 2>&1
ls -la $O
