timeout -s KILL 900 python -m pytest tests/test_gpu_kv_variants.py -x -q > gpurun_out/pytest139_var.log 2>&1; echo var=$?
timeout -s KILL 600 python scripts/kv_variant_bench.py --config opt-175b > gpurun_out/kv_var139.jsonl 2>&1; echo bench=$?
timeout -s KILL 300 python scripts/kv_variant_bench.py --config tiny --layers 64 > gpurun_out/kv_var139_tiny.jsonl 2>&1
