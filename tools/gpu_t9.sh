mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t9_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t9_pytest.log
for i in 1 2; do
VI_TMA_EPI=0 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t9_bench_direct_$i.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t9_bench_tma_$i.log 2>&1
done
VI_PROFILE_MODE=3 timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/t9_bench_m3.log 2>&1
timeout 900 python tools/refined_live.py > gpurun_out/t9_refined.log 2>&1; echo "rc=$?" >> gpurun_out/t9_refined.log
