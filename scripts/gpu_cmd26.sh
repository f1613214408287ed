set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/pytest26.log 2>&1
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep > gpurun_out/bench26_fused.json 2> gpurun_out/bench26_fused.err
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep --step two > gpurun_out/bench26_two.json 2> gpurun_out/bench26_two.err
echo done
