python __graft_entry__.py smoke > gpurun_out/smoke92.log 2>&1; echo smoke=$?
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest92.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench92.json 2> gpurun_out/bench92.err; echo bench=$?
