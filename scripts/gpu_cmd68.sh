timeout -s KILL 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/var68.log 2>&1; echo t=$?
