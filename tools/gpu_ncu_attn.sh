cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_tc -s 3 -c 1 -o gpurun_out/ncu_ours python tools/attn_bench.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"flash|Flash|kernel" -s 3 -c 1 -o gpurun_out/ncu_fa4 python tools/attn_fa4.py > gpurun_out/ncu_fa4.log 2>&1
python tools/attn_fa4.py
ls -la gpurun_out/*.ncu-rep
