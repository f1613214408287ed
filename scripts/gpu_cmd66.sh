timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm66.log 2>&1; echo t=$?
for v in "" dqw16; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep66.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 66 144 >> gpurun_out/gemm_sweep66.txt 2>&1
done
FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so timeout -s KILL 200 python scripts/gemm_trace.py 1 144 > gpurun_out/trace66.txt 2>&1
echo done
