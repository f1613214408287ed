for c in tiny opt-6.7b; do timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 16 --reps 10; done
timeout -s KILL 120 python scripts/attn_sweep.py --config tiny --layers 64 --reps 10 --fused
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
