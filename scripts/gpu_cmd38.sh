set -x
for lib in libflexq.so libflexq_noquant.so libflexq_nocopy.so libflexq_nothing.so; do for f in "" --fused; do FLEXQ_LIB=paper_2303_06865_b200/$lib timeout -s KILL 120 python scripts/attn_sweep.py --config opt-175b --layers 6 $f | sed "s/^/$lib /" >> gpurun_out/sweep38.txt 2>&1; done; done
echo done
