cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2; do
for cfg in "new:" "old:$V/libdit_oldattn.so" "everywait:$V/libdit_everywait.so"; do
  n=${cfg%%:*}; lib=${cfg#*:}
  echo "== $n"; DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py 8 24 4608 128
done; done
