mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t12_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t12_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t12_bench.log 2>&1
timeout 300 python bench.py --config C3T1 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t12_bench_t1.log 2>&1
timeout 900 python tools/refined_live.py > gpurun_out/t12_refined.log 2>&1; echo "rc=$?" >> gpurun_out/t12_refined.log
timeout 600 python tools/context_sweep.py --steps 30 > gpurun_out/t12_sweep.log 2>&1
