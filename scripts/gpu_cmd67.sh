set -x
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest67.log 2>&1; echo t=$?
timeout -s KILL 600 python bench.py > gpurun_out/bench67.json 2> gpurun_out/bench67.err; echo b=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:dequant_gemm -s 1 -c 1 -o gpurun_out/gemm_full67 python scripts/gemm_sweep.py --only --m 144 --reps 1 > gpurun_out/ncu_gemm67.log 2>&1; echo n=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 16 64 144 160 > gpurun_out/gemm_sweep67.txt 2>&1
echo done
