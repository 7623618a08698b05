#!/bin/bash
# GPU test run: build, the GPU parity suite with the per-test error / bar log, smoke.
# usage (from gpurun): bash tools/gpu_tests.sh [pytest -k expr]
set -o pipefail
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -m paper_2403_16161_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
rm -f gpurun_out/parity_log.jsonl
K=()
[ -n "$1" ] && K=(-k "$1")
VI_PARITY_LOG=gpurun_out/parity_log.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 "${K[@]}" > gpurun_out/gpu_tests.log 2>&1
rc=$?
tail -40 gpurun_out/gpu_tests.log
exit $rc
