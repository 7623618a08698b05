set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t3_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tp.py -x -q > gpurun_out/t3_pytest_tp.log 2>&1; echo "rc=$?" >> gpurun_out/t3_pytest_tp.log
timeout 300 python bench.py --tp --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/t3_tp1_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 200 --csv --log-file gpurun_out/t3_tp1_launches.csv \
   python bench.py --tp --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/t3_tp1_ncu.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/t3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 102 -c 6 -o gpurun_out/t3_gemm \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/t3_ncu_gemm.log 2>&1
