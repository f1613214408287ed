set -x
python __graft_entry__.py smoke > gpurun_out/smoke45.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest45.log 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/bench45.json 2> gpurun_out/bench45.err
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench45_ref.json 2> gpurun_out/bench45_ref.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_attention|quantize" -c 400 --csv --log-file gpurun_out/launches45.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch45.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_full45 python scripts/attn_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_full45.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:decode_attention_kernel -s 2 -c 1 -o gpurun_out/attn_fused_full45 python scripts/attn_sweep.py --layers 2 --reps 1 --fused > gpurun_out/ncu_fused45.log 2>&1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:topk -s 2 -c 1 -o gpurun_out/topk_full45 python scripts/topk_sweep.py --layers 2 --reps 1 > gpurun_out/ncu_topk45.log 2>&1
echo done
