timeout -s KILL 900 python bench.py > gpurun_out/bench72.json 2> gpurun_out/bench72.err; echo b=$?
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench72_ref.json 2> gpurun_out/bench72_ref.err; echo r=$?
