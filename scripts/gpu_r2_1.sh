set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_fused or exact_ties" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.log; tail -3 gpurun_out/r2_bench0.log
