timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
FLEXQ_ATTN_SPLIT=0,0,0 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "attention" 2>&1 | tail -2
FLEXQ_ATTN_SPLIT=0,100,4 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "attention" 2>&1 | tail -2
for sp in "400,0,0" "0,0,0" "100000,0,0" "400,50,2" "400,100,2"; do
  for cfg in "opt-175b 0" "opt-175b 72" "opt-175b 36" "opt-175b 18" "opt-30b 0" "opt-6.7b 0"; do
    set -- $cfg
    echo -n "split $sp "; FLEXQ_ATTN_SPLIT=$sp timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6
  done
done
