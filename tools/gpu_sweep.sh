cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2; do for n in base mspin sspin bspin; do
  lib=$V/libdit_$n.so; [ $n = base ] && lib=
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4608 128 | tail -1)"
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4429 64 | tail -1)"
done; done
