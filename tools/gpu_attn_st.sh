cd $GRAFT_REPO_ROOT
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants
for r in 1 2; do
for v in base p6 p10 p16 r216 r200; do
  L=""; if [ $v != base ]; then L=$V/libdit_$v.so; fi
  echo "== $v run $r: $(DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 2>&1 | tail -1 | awk "{print \$8}") / d64: $(DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 8 24 4429 64 2>&1 | tail -1 | awk "{print \$8}")"
done
done
