timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > gpurun_out/p110.log 2>&1; echo t=$?
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-sweep --no-offload > gpurun_out/bench110.json 2>/dev/null; echo b=$?
