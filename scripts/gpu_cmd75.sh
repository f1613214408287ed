timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm75.log 2>&1; echo t=$?
for v in "" nodefer dqw8; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep75.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 >> gpurun_out/gemm_sweep75.txt 2>&1
done
FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so timeout -s KILL 200 python scripts/gemm_trace.py 1 144 > gpurun_out/trace75.txt 2>&1
