set -x
for cfg in 32,4 32,3 32,2 16,5 16,4 16,3 64,2; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep1.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention -s 2 -c 1 -o gpurun_out/attn_full python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full.log 2>&1
timeout -s KILL 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attention|quantize" -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch.log 2>&1
echo done
