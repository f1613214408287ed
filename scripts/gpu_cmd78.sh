timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -k "attention_parity or full_size" > gpurun_out/par78.log 2>&1; echo t=$?
