cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2; do
for n in old new; do
  lib=$V/libdit_oldgemm.so; [ $n = new ] && lib=
  echo "== $n"; DIT_LIB_OVERRIDE=$lib timeout 200 python tools/resid_bench.py 2>&1 | head -3
done; done
