cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
python -c "import json; d=json.load(open('gpurun_out/r2d_bench.json')); print(d['value'], d['clocks'], d['kernels']['attention'], d['roofline']['frac'])"
for w in sd3m sd35l cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2d_bench_$w.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r2d_bench_$w.json')); print('$w', d['value'], d['clocks']['sm_mhz'], d['kernels']['attention'])"; done
