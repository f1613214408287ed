FLEXQ_LIB=paper_2303_06865_b200/libflexq_abg2.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or extreme" > gpurun_out/fa109.log 2>&1; echo t=$?
for v in "" abg2 abg0 "" abg2; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/fa109.txt
  FLEXQ_LIB=$lib timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 --fused >> gpurun_out/fa109.txt 2>&1
done
