timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 64 144 2>&1 | cut -c1-110
