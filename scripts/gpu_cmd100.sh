timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "quantize or dequantize or append" > gpurun_out/q100.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/quant_sweep.py > gpurun_out/q100.txt 2>&1
