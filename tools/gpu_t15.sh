mkdir -p gpurun_out
for r in 1 2 3; do
echo -n "old: "; tools/micro/attn_micro_old 100 x 0 2
echo -n "new: "; tools/micro/attn_micro 100 x 0 2
done > gpurun_out/am5.log 2>&1
tools/micro/attn_micro 50 t 0 2 >> gpurun_out/am5.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t15_build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t15_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t15_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t15_bench.log 2>&1
timeout 300 python tools/online_vs_memory.py > gpurun_out/t15_ovm.log 2>&1
