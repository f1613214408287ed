set -x
for cfg in 64,2,2,4,576 64,2,1,4,576 64,2,3,4,576 64,2,2,8,576 64,2,2,4,1024 32,3,3,4,576 32,3,1,4,576 32,2,3,4,576 32,4,2,4,576; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep15.txt 2>&1; done
for cfg in 64,2,2,4,576 32,3,3,4,576; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config opt-30b --layers 4 >> gpurun_out/sweep15.txt 2>&1; FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config opt-6.7b --layers 8 >> gpurun_out/sweep15.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full15 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full15.log 2>&1
echo done
