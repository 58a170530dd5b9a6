cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for n in gtrace mlptr; do echo "== $n"; DIT_LIB_OVERRIDE=$V/libdit_$n.so python tools/gemm_trace.py | grep -A2 "^resid" ; done
for rep in 1 2; do for n in base mlp; do
  lib=$V/libdit_$n.so; [ $n = base ] && lib=
  echo "== $n"; DIT_LIB_OVERRIDE=$lib timeout 200 python tools/resid_bench.py 2>&1 | head -3
done; done
