set -x
python __graft_entry__.py smoke > gpurun_out/smoke14.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest14.log 2>&1
for cfg in 64,2,4,4,1024 64,2,2,4,576 64,3,4,4,576 32,3,4,4,576; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep14.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full14 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full14.log 2>&1
echo done
