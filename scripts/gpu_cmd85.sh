timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm85.log 2>&1; echo t=$?
for v in "" nodqbar; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep85.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 >> gpurun_out/gemm_sweep85.txt 2>&1
  FLEXQ_GEMM_PAIR=1 FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/gemm_sweep85.txt 2>&1
done
