mkdir -p gpurun_out
for r in 1 2; do
echo -n "old: "; tools/micro/attn_micro_old 100 x 0 2
echo -n "fix: "; tools/micro/attn_micro 100 x 0 2
done > gpurun_out/am6.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t16_build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t16_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t16_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t16_bench.log 2>&1
