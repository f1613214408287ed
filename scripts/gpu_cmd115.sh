python __graft_entry__.py smoke > gpurun_out/smoke115.log 2>&1; echo smoke=$?
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest115.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench115.json 2> gpurun_out/bench115.err; echo bench=$?
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:dequant_gemm -s 1 -c 1 -o gpurun_out/gemm_full115 python scripts/gemm_sweep.py --only --m 144 --reps 1 > gpurun_out/ncu_gemm115.log 2>&1; echo ncu=$?
timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 16 64 144 160 > gpurun_out/gemm_sweep115.txt 2>&1
