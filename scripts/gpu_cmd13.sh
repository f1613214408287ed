set -x
python __graft_entry__.py smoke > gpurun_out/smoke13.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest13.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks13.csv &
CLK=$!
timeout -s KILL 600 python bench.py > gpurun_out/bench13.json 2> gpurun_out/bench13.err
kill $CLK
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench13_ref.json 2> gpurun_out/bench13_ref.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -c 400 --csv --log-file gpurun_out/launches13.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch13.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full13 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full13.log 2>&1
echo done
