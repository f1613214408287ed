set -x
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_nf25 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu25a.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_f25 python scripts/attn_sweep.py --layers 2 --reps 1 --fused > gpurun_out/ncu25b.log 2>&1
echo done
