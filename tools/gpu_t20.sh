mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t20_build.log 2>&1 || exit 1
for c in C4 C2 C3T1; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t20_bench_$c.log 2>&1; done
timeout 300 python bench.py --tp --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/t20_bench_tp1.log 2>&1
