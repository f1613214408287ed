timeout -s KILL 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sanitizer.py -q -x 2>&1 | grep -v "^\s*$" | tail -40
