# k-block lockstep experiment: cfg3 bench at several leads, then ncu DRAM bytes per GEMM type
cd $GRAFT_REPO_ROOT
O=gpurun_out/lock2
mkdir -p $O
DIT_GEMM_LOCK_D=16 timeout 600 python -m pytest tests/test_gpu_gemm_lock.py -x -q > $O/pytest_lock.log 2>&1; tail -2 $O/pytest_lock.log
for r in 1 2; do
for d in -1 16 64; do
  echo "== DIT_GEMM_LOCK_D=$d run $r"
  DIT_GEMM_LOCK_D=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b_${d}_$r.json 2>$O/b_${d}_$r.err
  python tools/bench_brief.py $O/b_${d}_$r.json
done
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for d in 16; do
DIT_GEMM_LOCK_D=$d timeout 900 ncu --metrics $M --clock-control none -k regex:gemm_kernel -c 612 --csv --log-file $O/traffic_$d.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
echo "ncu rc $?"
done
