#!/bin/bash
# DRAM bytes + duration of the fc2 (gemm launch 8) and linear2 (gemm launch 156) launches of one step,
# for the rasterisation-group variants built by tools/variant.py (g4, g6, g8, g32) and the default.
cd $GRAFT_REPO_ROOT
for v in base g4 g6 g8 g32; do
  L=paper_2604_08123_b200/build/variants/libdit_$v.so; [ $v = base ] && L=""
  for idx in 8 156; do
    DIT_LIB_OVERRIDE=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:gemm -s $idx -c 1 python tools/profile_step.py --steps 1 2>/dev/null | \
      grep -E "duration|dram__bytes|tensor" | awk -v v=$v -v i=$idx '{printf "%s %s %s %s %s\n", v, i, $1, $(NF-1), $NF}'
  done
done
