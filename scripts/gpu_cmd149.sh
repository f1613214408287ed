for c in opt-30b opt-6.7b; do
  timeout -s KILL 600 python bench.py --config $c --no-sweep --no-offload --no-cpu-baseline > gpurun_out/bench149_$c.json 2>/dev/null; echo $c=$?
done
