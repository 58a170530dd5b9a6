cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_lora_async.py tests/test_gpu_merge.py tests/test_gpu_plan_events.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_graph.json 2>gpurun_out/bench_graph.err; tail -3 gpurun_out/bench_graph.err
python -c "
import json; d=json.load(open('gpurun_out/bench_graph.json')); print(d['value'], d['ms_per_step'], d['graph'], d['e2e'], d['clocks'])"
timeout 300 python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_graph2.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_graph2.json')); print(d['value'], d['ms_per_step'], d['graph'])"
