set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k topk > gpurun_out/pytest19.log 2>&1
FLEXQ_LIB=paper_2303_06865_b200/libflexq_topk5.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k topk >> gpurun_out/pytest19.log 2>&1
for lib in libflexq.so libflexq_topk5.so; do for c in opt-175b opt-30b; do FLEXQ_LIB=paper_2303_06865_b200/$lib timeout -s KILL 120 python scripts/topk_sweep.py --config $c | sed "s/^/$lib /" >> gpurun_out/topk19.txt 2>&1; done; done
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:topk -s 2 -c 1 -o gpurun_out/topk_full19 python scripts/topk_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_topk19.log 2>&1
echo done
