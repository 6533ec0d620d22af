mkdir -p gpurun_out/r02ring
P=gpurun_out/r02ring
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_RK64=7_BLADE_ATTN2P_RV64=5.so" "libblade_asa_BLADE_ATTN2P_RK64=5_BLADE_ATTN2P_RV64=7.so" "libblade_asa_BLADE_ATTN2P_RK64=8_BLADE_ATTN2P_RV64=4.so"; do
  BLADE_LIB=$lib timeout 120 python scripts/attn_time.py --workload cog --calls 40 --blocks 2 >> $P/cog.jsonl 2>&1
done
done
grep -h median $P/cog.jsonl | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['lib'], d['ms'])
"
