set -x
for lib in libflexq.so libflexq_vidp.so; do for c in opt-175b opt-30b opt-6.7b; do FLEXQ_LIB=paper_2303_06865_b200/$lib timeout -s KILL 120 python scripts/attn_sweep.py --config $c --layers 6 | sed "s/^/$lib /" >> gpurun_out/sweep32.txt 2>&1; done; done
echo done
