set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest7.log 2>&1
for cfg in 64,2,4,2 64,2,4,1 64,2,4,4 64,2,4,8 64,3,4,2 32,3,4,2 32,2,4,2 32,2,4,4 32,4,4,2; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 >> gpurun_out/sweep7.txt 2>&1; done
echo done
