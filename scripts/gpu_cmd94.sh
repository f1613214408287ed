timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_offload.py tests/test_gpu_sanitizer.py -q -x > gpurun_out/pdl94.log 2>&1; echo t=$?
for pdl in 1 0 1 0; do
  FLEXQ_PDL=$pdl timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-sweep --no-offload > gpurun_out/bench94_pdl$pdl.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench94_pdl$pdl.json').read()); print('pdl=$pdl', d['ms_per_step'], d['value'], d['roofline']['us_per_launch'], d['clocks']['sm_mhz'])" >> gpurun_out/pdl94.txt
done
