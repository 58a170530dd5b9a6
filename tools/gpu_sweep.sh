cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2 3; do for n in withtrace new; do
  lib=$V/libdit_$n.so; [ $n = new ] && lib=
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4608 128 | tail -1)"
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4429 64 | tail -1)"
done; done
DIT_LIB_OVERRIDE=$V/libdit_trace.so TRACE=1 python tools/attn_bench.py | tail -3
timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "attention or head_dim" 2>&1 | tail -2
