set -x
python __graft_entry__.py smoke > gpurun_out/smoke3.log 2>&1
timeout -s KILL 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest3.log 2>&1
for cfg in 32,2,4 32,3,4 32,3,5 64,2,4 16,4,4; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep3.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention -s 2 -c 1 -o gpurun_out/attn_full3 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full3.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none -k regex:quantize -s 1 -c 2 -o gpurun_out/quant_full3 python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_quant3.log 2>&1
echo done
