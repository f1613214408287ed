for v in "" stp1 stp2 abg0 "" stp1 stp2; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/fa111.txt
  FLEXQ_LIB=$lib timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 --fused >> gpurun_out/fa111.txt 2>&1
done
