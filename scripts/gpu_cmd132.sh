for t in default topk_w2m8 topk_w4m4 topk_w2m6 topk_w3m5; do
  if [ "$t" = default ]; then unset FLEXQ_LIB; else export FLEXQ_LIB=$PWD/paper_2303_06865_b200/libflexq_$t.so; fi
  for c in opt-175b opt-30b; do timeout -s KILL 120 python scripts/topk_sweep.py --config $c --layers 4 | sed "s/^/$t /"; done
done
unset FLEXQ_LIB
