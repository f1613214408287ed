set -x
python __graft_entry__.py smoke > gpurun_out/smoke4.log 2>&1
timeout -s KILL 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest4.log 2>&1
for cfg in 32,2,4 32,3,4 32,3,5 32,4,4; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep4.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention -s 2 -c 1 -o gpurun_out/attn_full4 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full4.log 2>&1
echo done
