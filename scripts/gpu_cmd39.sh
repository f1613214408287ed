set -x
for rep in 1 2; do for lib in libflexq.so libflexq_nofence.so libflexq_nogstore.so libflexq_noquant.so; do FLEXQ_LIB=paper_2303_06865_b200/$lib timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 6 --fused | sed "s/^/$lib /" >> gpurun_out/sweep39.txt 2>&1; done; done
echo done
