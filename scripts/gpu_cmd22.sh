set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or attention_parity or topk" > gpurun_out/pytest22.log 2>&1
for f in "" --fused; do for c in opt-175b opt-30b opt-6.7b; do timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 $f >> gpurun_out/sweep22.txt 2>&1; done; done
echo done
