export FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so
for cfg in "opt-175b 0" "opt-6.7b 0"; do
  set -- $cfg
  FLEXQ_PDL=0 timeout 300 python scripts/attn_trace.py --config $1 --batch $2 --layers 4
  FLEXQ_PDL=0 timeout 300 python scripts/attn_trace.py --config $1 --batch $2 --layers 4
done
