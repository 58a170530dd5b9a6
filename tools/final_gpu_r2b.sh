set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2final5
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu,driver_version --format=csv > $O/nvsmi.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for w in cfg2 cfg4 cfg5 sd3m sd35l; do timeout 400 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2>/dev/null; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 2 -c 1 -o $O/attn_cfg3 python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 154 -c 1 -o $O/gemm_l1_cfg3 python tools/profile_step.py --steps 1 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
ls -la $O
