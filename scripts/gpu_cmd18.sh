set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k topk > gpurun_out/pytest18.log 2>&1
timeout -s KILL 120 python scripts/topk_sweep.py > gpurun_out/topk18.txt 2>&1
timeout -s KILL 120 python scripts/topk_sweep.py --config opt-30b >> gpurun_out/topk18.txt 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:topk -s 2 -c 1 -o gpurun_out/topk_full18 python scripts/topk_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_topk18.log 2>&1
echo done
