mkdir -p gpurun_out/r02split4
P=gpurun_out/r02split4
L="libblade_asa_BLADE_ATTN2P_SPLIT64=1_BLADE_ATTN2P_SEPP=1.so"
BLADE_LIB=$L timeout 60 python scripts/split_check.py > $P/check.log 2>&1; echo "rc=$?" >> $P/check.log; cat $P/check.log
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_SEPP=1.so" "$L"; do
  BLADE_LIB=$lib timeout 120 python scripts/attn_time.py --workload cog --calls 50 --blocks 3 >> $P/cog.jsonl 2>&1
done
done
grep -h median $P/cog.jsonl
