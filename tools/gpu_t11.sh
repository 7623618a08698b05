mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t11_build.log 2>&1 || exit 1
for v in "VI_ATTN_SK=2" "VI_ATTN_SK=1" "VI_ATTN_SK=3" "VI_ATTN_SPLIT=1" "VI_ATTN_SPLIT=1 VI_ATTN_COLSPLIT=1"; do
  echo -n "[$v] " >> gpurun_out/t11_t1.log
  env $v timeout 300 python bench.py --config C3T1 --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['value']), round(d['roofline']['avg_launch_ms']*1e3,2), d['device_time_ms_per_step'])" >> gpurun_out/t11_t1.log
done
