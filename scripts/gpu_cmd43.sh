set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/pytest43.log 2>&1
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep --no-e2e > gpurun_out/bench43_fused.json 2> gpurun_out/bench43_fused.err
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep --no-e2e --step two > gpurun_out/bench43_two.json 2> gpurun_out/bench43_two.err
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep --no-e2e > gpurun_out/bench43_fused2.json 2> gpurun_out/bench43_fused2.err
timeout -s KILL 600 python bench.py --steps 16 --no-cpu-baseline --no-sweep --no-e2e --step two > gpurun_out/bench43_two2.json 2> gpurun_out/bench43_two2.err
echo done
