timeout -s KILL 900 python bench.py --no-sweep --no-offload --no-cpu-baseline > gpurun_out/bench98.json 2> gpurun_out/bench98.err; echo b=$?
timeout -s KILL 900 python bench.py --no-sweep --no-offload --no-cpu-baseline --step two > gpurun_out/bench98_two.json 2> gpurun_out/bench98_two.err; echo b2=$?
