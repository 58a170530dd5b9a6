cd $GRAFT_REPO_ROOT
timeout 120 python tools/resid_bench.py 2>&1 | head -3
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -4
for rep in 1 2; do for cl in 2 4; do
  echo "== cl$cl $(DIT_GEMM_CL=$cl timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["clocks"]["sm_mhz"], round(d["kernels"]["gemm"]["tflops"]), {k:round(v["tflops"]) for k,v in d["kernels"]["gemm_by_type"].items()})')"
done; done
