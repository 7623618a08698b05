set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t2_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tp.py -x -q > gpurun_out/t2_pytest_tp.log 2>&1; echo "rc=$?" >> gpurun_out/t2_pytest_tp.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t2_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t2_bench.log 2>&1
timeout 300 python bench.py --tp --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t2_bench_tp1.log 2>&1
