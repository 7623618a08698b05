mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t8_build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_refined.py -x -q > gpurun_out/t8_pytest_ref.log 2>&1; echo "rc=$?" >> gpurun_out/t8_pytest_ref.log
timeout 900 python tools/refined_live.py > gpurun_out/t8_refined.log 2>&1; echo "rc=$?" >> gpurun_out/t8_refined.log
