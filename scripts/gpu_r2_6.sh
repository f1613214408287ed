timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for sp in "0,1" "100,2" "100,4" "50,2"; do
  for cfg in "opt-175b 0" "opt-175b 18" "opt-6.7b 0"; do
    set -- $cfg
    echo "split $sp"; FLEXQ_ATTN_SPLIT=$sp timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6
  done
done
