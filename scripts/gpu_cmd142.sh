timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 16 64 144 160 2>&1 | cut -c1-60 | sed 's/^/single /'
FLEXQ_GEMM_PAIR=1 timeout -s KILL 300 python scripts/gemm_sweep.py --m 1 16 64 144 160 2>&1 | cut -c1-60 | sed 's/^/pair   /'
