timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest69.log 2>&1; echo t=$?
timeout -s KILL 300 python scripts/quant_sweep.py --variants > gpurun_out/quant_var69.txt 2>&1; echo s=$?
python __graft_entry__.py smoke > gpurun_out/smoke69.log 2>&1; echo smoke=$?
