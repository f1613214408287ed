for v in "" nometa; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep91.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/gemm_sweep91.txt 2>&1
  FLEXQ_GEMM_PAIR=1 FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/gemm_sweep91.txt 2>&1
done
