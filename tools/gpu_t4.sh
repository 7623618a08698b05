set -x
mkdir -p gpurun_out
tools/micro/attn_micro 50 t 0 3 > gpurun_out/am2.log 2>&1
tools/micro/attn_micro 50 x 0 2 >> gpurun_out/am2.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t4_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t4_pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t4_bench.log 2>&1
