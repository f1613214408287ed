set -x
timeout -s KILL 240 python -m pytest tests/test_gpu_gemm.py -x -q -k "m1_one_tile" > gpurun_out/gemm48a.log 2>&1; echo a=$?
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q > gpurun_out/gemm48.log 2>&1; echo b=$?
echo done
