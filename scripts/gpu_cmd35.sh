set -x
for u in 1 2 3 4 6 8; do FLEXQ_UNITS_PER_WARP=$u timeout -s KILL 120 python scripts/attn_sweep.py --config opt-6.7b --layers 8 | sed "s/^/upw=$u /" >> gpurun_out/sweep35.txt 2>&1; done
for u in 1 2 3 4; do FLEXQ_UNITS_PER_WARP=$u timeout -s KILL 120 python scripts/attn_sweep.py --config opt-30b --layers 6 | sed "s/^/upw=$u /" >> gpurun_out/sweep35.txt 2>&1; done
for cfg in 64,2,3,4,1088 64,2,2,4,1024 64,2,4,4,1024 64,2,2,4,576 32,3,3,4,576; do for c in opt-30b opt-6.7b opt-175b; do FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 >> gpurun_out/sweep35.txt 2>&1; done; done
echo done
