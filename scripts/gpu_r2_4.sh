timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/r2_attn_fused_full python scripts/attn_sweep.py --layers 2 --reps 1 --fused > /dev/null 2>&1
ls -la gpurun_out/
