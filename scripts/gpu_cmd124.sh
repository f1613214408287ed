# in-step (power-capped) comparison of attention stage geometries: the bench step alone
for cfg in default 64,2,1,4,576 64,2,3,4,576 32,3,3,4,576 32,4,2,4,576 64,2,2,8,576; do
  if [ "$cfg" = default ]; then unset FLEXQ_ATTN_CFG; else export FLEXQ_ATTN_CFG=$cfg; fi
  timeout -s KILL 300 python bench.py --no-sweep --no-offload --no-cpu-baseline --no-e2e > gpurun_out/step124_$cfg.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/step124_$cfg.json')); r=d['roofline']; print('$cfg', d['ms_per_step'], d['value'], r['us_per_launch'], r['frac'], d['clocks']['sm_mhz'])"
done
