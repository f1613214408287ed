for p in 0 1 2 4 6; do
  FLEXQ_GEMM_PARTS=$p timeout -s KILL 120 python scripts/gemm_sweep.py --m 1 144 --shapes 12288x12288 2>&1 | sed "s/^/parts=$p /"
done
