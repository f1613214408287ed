set -x
timeout -s KILL 240 python -m pytest tests/test_gpu_gemm.py -q -x -k "m1_one_tile or pack_weight" > gpurun_out/gemm52a.log 2>&1; echo a=$?
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q > gpurun_out/gemm52.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 64 144 160 > gpurun_out/gemm_sweep52.txt 2>&1; echo s=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:dequant_gemm -s 1 -c 1 -o gpurun_out/gemm_full52 python scripts/gemm_sweep.py --only --reps 1 > gpurun_out/ncu_gemm52.log 2>&1; echo n=$?
echo done
