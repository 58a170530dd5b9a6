cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
timeout 1200 python -m pytest -q -p no:cacheprovider tests -m gpu 2>&1 | tail -3
for n in base otma0 base otma0 base otma0; do
  lib=$V/libdit_$n.so; [ $n = base ] && lib=
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["clocks"]["sm_mhz"], round(d["kernels"]["gemm"]["tflops"]), {k:round(v["tflops"]) for k,v in d["kernels"]["gemm_by_type"].items() if k in ("dbl_fc1","sgl_linear1","dbl_qkv","dbl_proj")})')"
done
