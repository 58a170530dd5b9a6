cd $GRAFT_REPO_ROOT
for h in 0 1 0 1; do
  echo "== DIT_GROUP_HEAVY=$h"
  DIT_GROUP_HEAVY=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/grp_$h.json 2>/dev/null
  python tools/bench_brief.py gpurun_out/grp_$h.json
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for h in 1 0; do
DIT_GROUP_HEAVY=$h timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 612 --csv --log-file gpurun_out/gemm_traffic_cfg3_h$h.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
echo "ncu rc $?"
done
