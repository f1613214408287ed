timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -5
timeout 1200 python bench.py > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.log; tail -3 gpurun_out/r2_bench3.log
