timeout -s KILL 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sanitizer.py -q -x 2>&1 | tail -1
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 64 144 160 2>&1 | cut -c1-60
