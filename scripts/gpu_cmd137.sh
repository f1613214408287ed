python __graft_entry__.py smoke > gpurun_out/smoke137.log 2>&1; echo smoke=$?
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest137.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench137.json 2> gpurun_out/bench137.err; echo bench=$?
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench137_ref.json 2> gpurun_out/bench137_ref.err; echo ref=$?
