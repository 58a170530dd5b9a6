cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_merge.py tests/test_gpu_lora_async.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/merge_bench.py 2>&1 | tail -4
