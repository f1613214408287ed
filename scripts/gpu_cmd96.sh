for cfg in "" "64,2,1,4,576" "64,2,3,4,576" "32,3,3,4,576" "32,3,1,4,576" "32,2,3,4,576" "32,4,2,4,576" "64,2,4,4,1024" "64,2,2,8,576"; do
  echo "== $cfg" >> gpurun_out/sweep96.txt
  FLEXQ_ATTN_CFG=$cfg timeout -s KILL 120 python scripts/attn_sweep.py --config opt-6.7b --layers 16 >> gpurun_out/sweep96.txt 2>&1
done
