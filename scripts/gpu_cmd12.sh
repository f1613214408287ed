set -x
for lib in libflexq.so libflexq_kidp4a.so libflexq_h16unpack.so; do for cfg in 64,2,4,4,1024 64,2,2,4,576; do FLEXQ_LIB=paper_2303_06865_b200/$lib FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --layers 8 | sed "s/^/$lib /" >> gpurun_out/sweep12.txt 2>&1; done; done
FLEXQ_LIB=paper_2303_06865_b200/libflexq_kidp4a.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest12_idp.log 2>&1
FLEXQ_LIB=paper_2303_06865_b200/libflexq_kidp4a.so timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full12_idp python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full12.log 2>&1
echo done
