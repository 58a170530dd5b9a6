cd $GRAFT_REPO_ROOT
O=gpurun_out/bis
mkdir -p $O
T="tests/test_gpu_bmax16.py::test_sequence_parallel_sixteen_sequences_bitwise"
run() { name=$1; shift; timeout 300 python -m pytest "$@" -x -q -p no:cacheprovider > $O/$name.log 2>&1; echo "$name: $(tail -1 $O/$name.log)"; }
run full_order tests -m gpu -k "split or bmax16"
run s1 "tests/test_gpu_attn_split.py::test_split_tail_vs_torch_fp32[1-3-16896-128]" $T
run s4 tests/test_gpu_attn_split.py::test_split_tail_vs_torch_fp32 $T
run s5 tests/test_gpu_attn_split.py::test_split_tail_dit_step_vs_oracle $T
run all_then_T tests/test_gpu_attn_split.py $T
