python __graft_entry__.py smoke > gpurun_out/smoke140.log 2>&1; echo smoke=$?
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest140.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench140.json 2> gpurun_out/bench140.err; echo bench=$?
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench140_ref.json 2> gpurun_out/bench140_ref.err; echo ref=$?
