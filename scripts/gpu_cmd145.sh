python __graft_entry__.py smoke 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sanitizer.py -q 2>&1 | tail -1
