mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t24_build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t24_pytest.log
timeout 600 python bench.py > gpurun_out/t24_bench.log 2>&1
