set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py smoke > gpurun_out/smoke47.log 2>&1; echo smoke=$?
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest47.log 2>&1; echo pytest=$?
timeout -s KILL 600 python bench.py > gpurun_out/bench47.json 2> gpurun_out/bench47.err; echo bench=$?
echo done
