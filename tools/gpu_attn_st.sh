cd $GRAFT_REPO_ROOT
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants
for r in 1 2; do
for v in base pm7 pm5 pm6 pm2; do
  if [ $v = base ]; then L=""; else L=$V/libdit_$v.so; fi
  echo "== $v run $r"
  DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 2>&1 | tail -1
  DIT_LIB_OVERRIDE=$L timeout 120 python tools/attn_bench.py 8 24 4608 64 2>&1 | tail -1
done
done
