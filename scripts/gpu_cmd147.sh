FLEXQ_GEMM_PAIR=1 timeout -s KILL 600 compute-sanitizer --tool racecheck --kernel-name kns=dequant_gemm python scripts/sanitize_case.py 2>&1 | tail -8
FLEXQ_GEMM_PAIR=1 timeout -s KILL 600 python -m pytest tests/test_gpu_gemm.py -q 2>&1 | tail -1
