cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2; do for n in base rb0 rb1; do
  lib=$V/libdit_$n.so; [ $n = base ] && lib=
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4608 128 | tail -1)"
done; done
for n in base rb0; do lib=$V/libdit_$n.so; [ $n = base ] && lib=; DIT_LIB_OVERRIDE=$lib TRACE=1 python tools/attn_bench.py | tail -3; done
