timeout -s KILL 600 python -m pytest tests/test_gpu_kv_variants.py -q -k "wide or extreme or full_size" > gpurun_out/pytest136.log 2>&1; echo rc=$?
