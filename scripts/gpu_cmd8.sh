set -x
for cfg in 64,2,4,4,1024 64,2,2,4,576 64,2,1,4,576 64,2,4,4,576 32,2,4,4,576 32,3,2,4,576 64,2,4,8,1024; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep8.txt 2>&1; done
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest8.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err
echo done
