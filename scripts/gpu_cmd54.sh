for v in "" deqskip nomma ps12 nomma12; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep54.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/gemm_sweep54.txt 2>&1
done
echo done
