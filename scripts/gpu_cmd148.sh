python __graft_entry__.py smoke > gpurun_out/smoke148.log 2>&1; echo smoke=$?
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest148.log 2>&1; echo pytest=$?
