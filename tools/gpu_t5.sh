set -x
mkdir -p gpurun_out
tools/micro/attn_micro_88 50 t 0 3 > gpurun_out/am3.log 2>&1
for m in 92 AA; do tools/micro/attn_micro_$m 50 x 0 3 >> gpurun_out/am3.log 2>&1; done
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t5_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t5_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t5_bench.log 2>&1
