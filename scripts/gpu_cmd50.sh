set -x
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm50.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 16 64 144 256 > gpurun_out/gemm_sweep50.txt 2>&1; echo s=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:dequant_gemm -s 1 -c 1 -o gpurun_out/gemm_full50 python scripts/gemm_sweep.py --only --reps 1 > gpurun_out/ncu_gemm50.log 2>&1; echo n=$?
echo done
