#!/bin/bash
# Round evidence, in two gpurun calls (one ncu run per call):
#   bash tools/gpu_final.sh main   GPU tests (+ parity log), smoke, bench lines (C3 default with
#                                  cpu baseline; C3T1, C2, C4), the reference arm, ncu launch list
#   bash tools/gpu_final.sh attn   ncu --set full capture of the attention
# Outputs under gpurun_out/final/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { cat $O/build.log; exit 1; }
if [ "${1:-main}" = "main" ]; then
  VI_PARITY_LOG=$O/parity_log.jsonl timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
  timeout 900 python bench.py > $O/bench_C3.jsonl 2> $O/bench_C3.err; echo "bench rc=$?"
  for c in C3T1 C2 C4; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.jsonl 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc=$?"
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 700 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
else
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_attn.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sk2 -s 40 -c 2 \
    -o $O/attn_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
ls $O
