mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t19_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "window" > gpurun_out/t19_pytest_win.log 2>&1; echo "rc=$?" >> gpurun_out/t19_pytest_win.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t19_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t19_pytest.log
