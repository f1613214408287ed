timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sanitizer.py -q > gpurun_out/g114.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 > gpurun_out/g114.txt 2>&1
FLEXQ_GEMM_PAIR=1 timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/g114.txt 2>&1
