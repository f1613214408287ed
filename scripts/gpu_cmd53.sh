set -x
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/gemm53.log 2>&1; echo t=$?
for v in "" dqw8 deqskip; do
  lib=paper_2303_06865_b200/libflexq${v:+_$v}.so
  echo "== $v" >> gpurun_out/gemm_sweep53.txt
  FLEXQ_LIB=$lib timeout -s KILL 300 python scripts/gemm_sweep.py --only --m 1 64 144 >> gpurun_out/gemm_sweep53.txt 2>&1
done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:dequant_gemm -s 1 -c 1 -o gpurun_out/gemm_full53 python scripts/gemm_sweep.py --only --reps 1 > gpurun_out/ncu_gemm53.log 2>&1; echo n=$?
echo done
