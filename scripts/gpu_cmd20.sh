set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or attention_parity or append" > gpurun_out/pytest20.log 2>&1
for f in "" --fused; do for c in opt-175b opt-30b opt-6.7b; do timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 $f >> gpurun_out/sweep20.txt 2>&1; done; done
timeout -s KILL 600 python bench.py --steps 8 --no-cpu-baseline --no-sweep > gpurun_out/bench20_fused.json 2> gpurun_out/bench20_fused.err
timeout -s KILL 600 python bench.py --steps 8 --no-cpu-baseline --no-sweep --step two > gpurun_out/bench20_two.json 2> gpurun_out/bench20_two.err
echo done
