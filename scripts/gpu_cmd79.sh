timeout -s KILL 120 python -m pytest tests/test_gpu_gemm.py -q -x -k "m5_two_tiles" > gpurun_out/pair79a.log 2>&1; echo a=$?
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q > gpurun_out/pair79.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 160 > gpurun_out/gemm_sweep79.txt 2>&1; echo s=$?
FLEXQ_GEMM_PAIR=0 timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 > gpurun_out/gemm_sweep79_single.txt 2>&1
