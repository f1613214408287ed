set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest37.log 2>&1
for c in opt-175b opt-30b opt-6.7b; do timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 >> gpurun_out/sweep37.txt 2>&1; timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 --fused >> gpurun_out/sweep37.txt 2>&1; done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks37.csv &
CLK=$!
timeout -s KILL 600 python bench.py > gpurun_out/bench37.json 2> gpurun_out/bench37.err
kill $CLK
echo done
