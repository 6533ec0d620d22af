mkdir -p gpurun_out/r02pc3
P=gpurun_out/r02pc3
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv > $P/smi.txt
for rep in 1 2 3 4; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_PCHUNK=2.so"; do
  BLADE_LIB=$lib timeout 120 python scripts/attn_time.py --workload wan --calls 30 --blocks 2 >> $P/wan.jsonl 2>&1
  BLADE_LIB=$lib timeout 120 python scripts/attn_time.py --workload wan --calls 30 --blocks 2 --fused >> $P/wan_fused.jsonl 2>&1
done
done
cat $P/smi.txt; grep -h median $P/wan.jsonl $P/wan_fused.jsonl
