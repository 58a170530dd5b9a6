cd $GRAFT_REPO_ROOT
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants
for r in 1 2; do
for v in base v3d64 v3k2d64 pm7d64; do
  L=""; if [ $v != base ]; then L=$V/libdit_$v.so; fi
  echo "== $v run $r: d64 4429 $(DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 8 24 4429 64 2>&1 | tail -1 | awk "{print \$8}") / d64 4608 $(DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 8 24 4608 64 2>&1 | tail -1 | awk "{print \$8}")"
done
done
