timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for cfg in "opt-175b 0" "opt-175b 72" "opt-175b 36" "opt-175b 18" "opt-30b 0" "opt-6.7b 0" "tiny 0"; do
  set -- $cfg
  timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6
done
for sp in "0,1" "50,4" "100,2" "100,4" "100,8" "200,4"; do
  for cfg in "opt-175b 0" "opt-175b 18" "opt-6.7b 0"; do
    set -- $cfg
    echo "split $sp"; FLEXQ_ATTN_SPLIT=$sp timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6
  done
done
export FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so
for cfg in "opt-175b 0" "opt-6.7b 0"; do
  set -- $cfg
  FLEXQ_PDL=0 timeout 300 python scripts/attn_trace.py --config $1 --batch $2 --layers 4
done
