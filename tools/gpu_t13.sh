mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t13_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tp.py tests/test_gpu_parity.py -q > gpurun_out/t13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t13_pytest.log
timeout 300 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t13_bench_c2.log 2>&1
