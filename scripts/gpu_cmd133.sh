timeout -s KILL 900 python -m pytest tests/test_gpu_kv_variants.py tests/test_gpu_sanitizer.py -q > gpurun_out/pytest133.log 2>&1; echo rc=$?
