timeout -s KILL 900 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/san77.log 2>&1; echo t=$?
