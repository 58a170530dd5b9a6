cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_lora_async.py tests/test_gpu_parity.py -q -m gpu -x -k "attention or lora or async" -p no:cacheprovider 2>&1 | tail -3
for v in 1 0; do
  echo "== DIT_ATTN_V1=$v"
  DIT_ATTN_V1=$v timeout 120 python tools/attn_bench.py 8 24 4608 128
  DIT_ATTN_V1=$v timeout 120 python tools/attn_bench.py 8 24 4429 64
  DIT_ATTN_V1=$v timeout 120 python tools/attn_bench.py 1 24 16896 128
done
