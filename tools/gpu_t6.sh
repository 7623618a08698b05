mkdir -p gpurun_out
for r in 1 2; do
for m in 00 88 92 AA B6 EE d2_AA d2_B6; do echo -n "$m: "; tools/micro/attn_micro_$m 100 x 0 3; done
echo -n "sk2: "; tools/micro/attn_micro_88 100 x 0 2
done
