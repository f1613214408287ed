timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_offload.py tests/test_gpu_sanitizer.py -q -x > gpurun_out/fa107.log 2>&1; echo t=$?
for i in 1 2; do timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 --fused >> gpurun_out/fa107.txt 2>&1; done
timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 8 >> gpurun_out/fa107.txt 2>&1
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-sweep --no-offload > gpurun_out/bench107.json 2>/dev/null; echo b=$?
