#!/bin/bash
# Build libdit from the repo root, then run the GPU parity tests + a short bench on a B200 via gpurun.
# usage: tools/gpucheck.sh <tag> [pytest -k expr]
set -e
cd /root/repo
python __graft_entry__.py | tail -1
TAG=${1:-chk}
K=${2:-}
KARG=""
if [ -n "$K" ]; then KARG="-k $K"; fi
timeout 2400 /usr/local/graft/bin/gpurun --timeout 900 -- "timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x $KARG 2>&1 | tail -3; timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; python tools/bench_brief.py gpurun_out/bench_$TAG.json" 2>&1 | tail -12
