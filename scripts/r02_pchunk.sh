mkdir -p gpurun_out/r02pc2
P=gpurun_out/r02pc2
for L in "libblade_asa_BLADE_ATTN2P_PCHUNK=2.so" "libblade_asa_BLADE_ATTN2P_PCHUNK=4.so"; do
  BLADE_LIB=$L timeout 60 python scripts/split_check.py >> $P/check.log 2>&1; echo "rc=$?" >> $P/check.log
done
cat $P/check.log
for rep in 1 2 3; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_PCHUNK=2.so" "libblade_asa_BLADE_ATTN2P_PCHUNK=4.so"; do
  BLADE_LIB=$lib timeout 120 python scripts/attn_time.py --workload wan --calls 30 --blocks 2 >> $P/wan.jsonl 2>&1
done
done
grep -h median $P/wan.jsonl
