set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/pytest42.log 2>&1
for rep in 1 2; do for f in "" --fused; do timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 6 $f >> gpurun_out/sweep42.txt 2>&1; done; done
for f in "" --fused; do timeout -s KILL 120 python scripts/attn_sweep.py --config opt-30b --layers 6 $f >> gpurun_out/sweep42.txt 2>&1; timeout -s KILL 120 python scripts/attn_sweep.py --config opt-6.7b --layers 6 $f >> gpurun_out/sweep40.txt 2>&1; done
echo done
