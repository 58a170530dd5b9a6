cd $GRAFT_REPO_ROOT
O=gpurun_out/lock6
mkdir -p $O
V=$GRAFT_REPO_ROOT/paper_2604_08123_b200/build/variants/libdit_lockstats.so
echo "== group16"; DIT_LIB_OVERRIDE=$V timeout 300 python tools/lock_bench.py 0 100000 16 64 256 2>&1 | tee $O/lb_g16.txt
echo "== heavy"; DIT_GEMM_HEAVY_GROUP=1 DIT_LIB_OVERRIDE=$V timeout 300 python tools/lock_bench.py 0 100000 16 64 2>&1 | tee $O/lb_h.txt
