timeout -s KILL 400 python -m pytest tests/test_gpu_offload.py -q -x > gpurun_out/off71.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/offload_bench.py > gpurun_out/offbench71.txt 2>&1; echo b=$?
timeout -s KILL 300 python scripts/offload_bench.py --layers 4 --gpu-batches 3 --batch 48 >> gpurun_out/offbench71.txt 2>&1; echo b=$?
