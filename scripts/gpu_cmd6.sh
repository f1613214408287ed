set -x
python __graft_entry__.py smoke > gpurun_out/smoke6.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest6.log 2>&1
for cfg in 64,2,4 32,3,4 32,2,4 64,3,3 64,3,4 64,2,2; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep6.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention -s 2 -c 1 -o gpurun_out/attn_full6 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full6.log 2>&1
echo done
