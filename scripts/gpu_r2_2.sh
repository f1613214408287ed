# parity of the rewritten dense attention, then the per-config sweep
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
for cfg in "opt-175b 0" "opt-175b 72" "opt-175b 36" "opt-175b 18" "opt-30b 0" "opt-6.7b 0" "tiny 0"; do
  set -- $cfg
  timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6
  timeout 300 python scripts/attn_sweep.py --config $1 --batch $2 --layers 6 --fused
done
