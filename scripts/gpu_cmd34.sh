set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest34.log 2>&1
FLEXQ_LIB=paper_2303_06865_b200/libflexq_vidp.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "attention_parity" >> gpurun_out/pytest34.log 2>&1
for lib in libflexq.so libflexq_vidp.so; do for c in opt-175b opt-30b opt-6.7b; do FLEXQ_LIB=paper_2303_06865_b200/$lib timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 | sed "s/^/$lib /" >> gpurun_out/sweep34.txt 2>&1; done; done
timeout -s KILL 120 python scripts/topk_sweep.py >> gpurun_out/sweep34.txt 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full34 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu34.log 2>&1
echo done
