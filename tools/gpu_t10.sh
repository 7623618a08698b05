mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t10_build.log 2>&1 || exit 1
for bn in "" "ffn1=256" "qkv=256" "qkv=256,ffn1=256" "embed=256" "back=128" "o=64,ffn2=64" "qkv=256,ffn1=256,o=64"; do
  echo -n "BN[$bn]: " >> gpurun_out/t10_bn.log
  VI_BN="$bn" VI_PROFILE_MODE=3 timeout 300 python bench.py --steps 60 --warmup 10 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['device_time_ms_per_step'])" >> gpurun_out/t10_bn.log
done
