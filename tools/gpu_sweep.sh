cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "attention_kernel" -x 2>&1 | tail -3
for rep in 1 2; do for q in 0 1; do
  echo "== q3=$q $(DIT_ATTN_Q3=$q timeout 120 python tools/attn_bench.py 8 24 4429 64 | tail -1)"
  echo "== q3=$q $(DIT_ATTN_Q3=$q timeout 120 python tools/attn_bench.py 2 24 16384 64 | tail -1)"
done; done
timeout 900 python -m pytest -q -p no:cacheprovider tests -m gpu -x 2>&1 | tail -3
