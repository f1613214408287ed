set -x
timeout -s KILL 600 python -m pytest tests -m gpu -q > gpurun_out/pytest9.log 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke9.log 2>&1

timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full9 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full9.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:quantize_kernel -s 1 -c 2 -o gpurun_out/quant_full9 python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_quant9.log 2>&1
echo done
