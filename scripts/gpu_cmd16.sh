set -x
python __graft_entry__.py smoke > gpurun_out/smoke16.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest16.log 2>&1
for cfg in 64,2,3,4,576 64,2,3,4,1088; do for c in opt-175b opt-30b opt-6.7b; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 >> gpurun_out/sweep16.txt 2>&1; done; done
timeout -s KILL 600 python bench.py > gpurun_out/bench16.json 2> gpurun_out/bench16.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --same-device --config opt-6.7b --layers 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/bench16_2rank.json 2> gpurun_out/bench16_2rank.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -s 480 -c 384 --csv --log-file gpurun_out/launches16.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch16.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full16 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full16.log 2>&1
echo done
