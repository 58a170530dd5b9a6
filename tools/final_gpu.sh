set -x
cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests_final.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
for w in cfg2 cfg4 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_final_$w.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 2 -c 1 -o gpurun_out/attn_final python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 154 -c 1 -o gpurun_out/gemm_l1_final python tools/profile_step.py --steps 1 > /dev/null 2>&1
ls -la gpurun_out | tail -20
