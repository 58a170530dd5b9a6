cd $GRAFT_REPO_ROOT
DIT_ATTN_SI=1 timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "attention or head_dim or ragged or tiny" -x 2>&1 | tail -3
for rep in 1 2 3; do for si in 0 1; do
  echo "== si=$si $(DIT_ATTN_SI=$si timeout 120 python tools/attn_bench.py 8 24 4608 128 | tail -1)"
  echo "== si=$si $(DIT_ATTN_SI=$si timeout 120 python tools/attn_bench.py 8 24 4429 64 | tail -1)"
done; done
