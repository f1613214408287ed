for u in 0 1 2 4 8; do
  for c in tiny opt-6.7b; do
    FLEXQ_UNITS_PER_WARP=$u timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 64 --reps 10 | sed "s/^/u=$u /"
  done
done
