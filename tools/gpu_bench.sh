#!/bin/bash
# GPU bench run: build, then bench.py (default C3 line) plus optional extra configs.
# usage (from gpurun): bash tools/gpu_bench.sh [tag] [extra bench args...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-b}; shift
python -m paper_2403_16161_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.jsonl 2> gpurun_out/bench_$tag.err
rc=$?
tail -c 3000 gpurun_out/bench_$tag.jsonl; tail -5 gpurun_out/bench_$tag.err
exit $rc
