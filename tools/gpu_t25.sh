mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t25_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t25_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t25_pytest.log
for w in 16 10 8 6; do
  VI_SK_TAIL_W=$w timeout 300 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/t25_bench_w$w.log 2>&1
done
