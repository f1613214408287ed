timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "dequant" > gpurun_out/deq76.log 2>&1; echo t=$?
for v in "" deq1 deq4n deq2; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/deq_sweep76.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/quant_sweep.py >> gpurun_out/deq_sweep76.txt 2>&1
done
