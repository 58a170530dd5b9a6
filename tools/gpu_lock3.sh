# K-heavy GEMM raster (one round = every N-tile of clusters/tiles_n M-panels) x k-block lockstep
cd $GRAFT_REPO_ROOT
O=gpurun_out/lock3
mkdir -p $O
for r in 1 2; do
for hv in 0 1; do
for d in -1 16; do
  echo "== DIT_GEMM_HEAVY_GROUP=$hv DIT_GEMM_LOCK_D=$d run $r"
  DIT_GEMM_HEAVY_GROUP=$hv DIT_GEMM_LOCK_D=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b_${hv}_${d}_$r.json 2>$O/b_${hv}_${d}_$r.err
  python tools/bench_brief.py $O/b_${hv}_${d}_$r.json
done
done
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for d in 16 -1; do
DIT_GEMM_HEAVY_GROUP=1 DIT_GEMM_LOCK_D=$d timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 612 --csv --log-file $O/traffic_h1_$d.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
echo "ncu rc $?"
done
