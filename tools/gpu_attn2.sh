cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for cfg in "base:" "splitld:$V/libdit_splitld.so"; do
  n=${cfg%%:*}; lib=${cfg#*:}
  echo "== v1 $n"
  for shape in "8 24 4608 128" "8 24 4429 64"; do DIT_ATTN_V1=1 DIT_LIB_OVERRIDE=$lib timeout 120 python tools/attn_bench.py $shape; done
done
echo "== v2 104/40"
for shape in "8 24 4608 128" "8 24 4429 64"; do DIT_LIB_OVERRIDE=$V/libdit_v2r104.so timeout 120 python tools/attn_bench.py $shape; done
echo "== v1 base again"
for shape in "8 24 4608 128" "8 24 4429 64"; do DIT_ATTN_V1=1 timeout 120 python tools/attn_bench.py $shape; done
