python __graft_entry__.py smoke > gpurun_out/smoke101.log 2>&1; echo smoke=$?
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest101.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench101.json 2> gpurun_out/bench101.err; echo bench=$?
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench101_ref.json 2> gpurun_out/bench101_ref.err; echo ref=$?
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -s 96 -c 200 --csv --log-file gpurun_out/launches101.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep --no-offload > gpurun_out/ncu_launch101.log 2>&1; echo ncu=$?
