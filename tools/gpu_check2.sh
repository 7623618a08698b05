mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t21_build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t21_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t21_pytest.log
for v in "VI_TMA_EPI=1" "VI_PAIR=0" "VI_TMA_EPI=0"; do
  for i in 1 2; do echo -n "[$v] " >> gpurun_out/t21_ab.log; env $v VI_PROFILE_MODE=3 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['device_time_ms_per_step'])" >> gpurun_out/t21_ab.log; done
done
