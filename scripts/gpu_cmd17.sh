set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "topk or parity" > gpurun_out/pytest17.log 2>&1
timeout -s KILL 120 python scripts/topk_sweep.py > gpurun_out/topk17.txt 2>&1
timeout -s KILL 120 python scripts/topk_sweep.py --config opt-30b >> gpurun_out/topk17.txt 2>&1
for c in opt-175b opt-6.7b; do timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 >> gpurun_out/sweep17.txt 2>&1; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:topk -s 2 -c 1 -o gpurun_out/topk_full17 python scripts/topk_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_topk17.log 2>&1
echo done
