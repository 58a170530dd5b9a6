cd $GRAFT_REPO_ROOT
V=paper_2604_08123_b200/build/variants
for rep in 1 2; do for n in base lnb7 ln7; do
  lib=$V/libdit_$n.so; [ $n = base ] && lib=
  echo "== $n $(DIT_LIB_OVERRIDE=$lib timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["clocks"]["sm_mhz"], "lnmod", round(d["kernels"]["lnmod"]["ms_per_step"],2))')"
done; done
DIT_LIB_OVERRIDE=$V/libdit_lnb7.so timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "tiny or ragged or batch" 2>&1 | tail -2
