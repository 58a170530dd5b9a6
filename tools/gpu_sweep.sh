cd $GRAFT_REPO_ROOT
for rep in 1 2; do for cfgv in "base:0:0" "g16B2:0:2" "g6B2:6:2" "g6A1B2:6:12" "g6:6:0"; do
  n=${cfgv%%:*}; rest=${cfgv#*:}; gm=${rest%%:*}; hi=${rest#*:}
  echo "== $n $(DIT_GEMM_HEAVY_GROUP=$gm DIT_GEMM_HEAVY_HINTS=$hi timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["clocks"]["sm_mhz"], round(d["kernels"]["gemm"]["tflops"]), {k:round(v["tflops"]) for k,v in d["kernels"]["gemm_by_type"].items() if k in ("sgl_linear2","dbl_fc2","sgl_linear1")})')"
done; done
