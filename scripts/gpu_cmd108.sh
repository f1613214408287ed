for v in "" abq0 abg0 abn0 abf0; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/fa108.txt
  FLEXQ_LIB=$lib timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 --fused >> gpurun_out/fa108.txt 2>&1
done
timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 >> gpurun_out/fa108.txt 2>&1
