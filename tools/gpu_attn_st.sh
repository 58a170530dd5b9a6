cd $GRAFT_REPO_ROOT
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants
for r in 1 2; do
for v in head new split; do
  L=""; S=0
  if [ $v = head ]; then L=$V/libdit_head.so; fi
  if [ $v = split ]; then S=1; fi
  echo "== $v run $r"
  DIT_ATTN_SPLIT_TAIL=$S DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 2>&1 | tail -1
  DIT_ATTN_SPLIT_TAIL=$S DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 8 24 4608 64 2>&1 | tail -1
  DIT_ATTN_SPLIT_TAIL=$S DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 1 3 16896 128 2>&1 | tail -1
  DIT_ATTN_SPLIT_TAIL=$S DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 1 24 4608 128 2>&1 | tail -1
done
done
