mkdir -p gpurun_out
timeout 120 tools/micro/gemm_micro > gpurun_out/gm3.log 2>&1; echo "rc=$?" >> gpurun_out/gm3.log
for r in 1 2; do echo -n "old: "; tools/micro/attn_micro_old 100 x 0 2; echo -n "fix: "; tools/micro/attn_micro 100 x 0 2; done > gpurun_out/am7.log 2>&1
