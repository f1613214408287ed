for v in "" fwd2 fwd3; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep82.txt
  FLEXQ_LIB=$lib timeout -s KILL 200 python -m pytest tests/test_gpu_gemm.py -q -x -k "m144_split_k or m5_two or full_size" >> gpurun_out/gemm_sweep82.txt 2>&1
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 144 >> gpurun_out/gemm_sweep82.txt 2>&1
done
