#!/bin/bash
# GEMM rasterisation group sweep: bench + per-launch DRAM bytes of 20 GEMM launches
for g in 16 4 8 32; do
  if [ $g = 16 ]; then L=""; else L=paper_2604_08123_b200/build/libdit_g$g.so; fi
  DIT_LIB_OVERRIDE=$L timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g$g.json 2>/dev/null
  echo "group $g: $(python tools/bench_brief.py gpurun_out/bench_g$g.json | head -1)"
  DIT_LIB_OVERRIDE=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm_kernel -s 300 -c 20 --csv --log-file gpurun_out/ncu_g$g.csv python tools/profile_step.py > /dev/null 2>&1
done
