set -x
for cfg in 64,2,2,4,576 64,2,3,4,576 64,2,2,4,1088 64,2,3,4,1088; do for u in 0 1 2 3; do for c in opt-175b opt-30b opt-6.7b; do FLEXQ_UNITS_PER_WARP=$u FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 | sed "s/^/upw=$u /" >> gpurun_out/sweep36.txt 2>&1; done; done; done
echo done
