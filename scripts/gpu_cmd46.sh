set -x
timeout -s KILL 300 python scripts/offload_probe.py > gpurun_out/offload46.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -s 96 -c 200 --csv --log-file gpurun_out/launches46.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch46.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -s 96 -c 200 --csv --log-file gpurun_out/launches46_two.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --step two > gpurun_out/ncu_launch46_two.log 2>&1
echo done
