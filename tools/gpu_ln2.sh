cd $GRAFT_REPO_ROOT
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants
for r in 1 2; do
for v in base ln6 ln7 ln9; do
  L=""; if [ $v != base ]; then L=$V/libdit_$v.so; fi
  DIT_LIB_OVERRIDE=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ln2_$v_$r.json 2>/dev/null
  echo "== $v run $r: $(python -c "import json;d=json.load(open('gpurun_out/ln2_$v_$r.json'));print(round(d['value'],4), round(d['kernels']['lnmod']['ms_per_step'],2), d['clocks']['sm_mhz'])")"
done
done
