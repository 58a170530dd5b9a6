cd $GRAFT_REPO_ROOT
DIT_ATTN_KERNEL=hr timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "attention or head_dim or ragged or tiny" 2>&1 | tail -3
for rep in 1 2; do for k in v8 hr; do
  echo "== $k $(DIT_ATTN_KERNEL=$k timeout 120 python tools/attn_bench.py 8 24 4608 128 | tail -1)"
  echo "== $k $(DIT_ATTN_KERNEL=$k timeout 120 python tools/attn_bench.py 8 24 4429 64 | tail -1)"
done; done
