cd $GRAFT_REPO_ROOT
O=gpurun_out/grp3
mkdir -p $O
for r in 1 2; do
for cfgp in "16 16" "16 8" "16 4" "8 8" "12 8"; do
  set -- $cfgp
  echo "== light $1 heavy $2 run $r"
  DIT_GEMM_GROUP_LIGHT=$1 DIT_GEMM_GROUP_HEAVY=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b_$1_$2_$r.json 2>/dev/null
  python tools/bench_brief.py $O/b_$1_$2_$r.json 2>/dev/null | head -1
done
done
