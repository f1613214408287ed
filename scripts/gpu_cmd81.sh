timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pair81.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 160 > gpurun_out/gemm_sweep81.txt 2>&1; echo s=$?
FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so timeout -s KILL 200 python scripts/gemm_trace.py 1 144 > gpurun_out/trace81.txt 2>&1
