set -x
timeout -s KILL 300 python scripts/quant_sweep.py > gpurun_out/quant44.txt 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"quantize" --csv --log-file gpurun_out/quant44_ncu.csv python scripts/quant_sweep.py > /dev/null 2>&1
echo done
