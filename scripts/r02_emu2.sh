# Exponential-emulation sweep of the persistent attention kernel (attention alone, interleaved)
mkdir -p gpurun_out/r02emu2
P=gpurun_out/r02emu2
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_EMU128=0x01.so" "libblade_asa_BLADE_ATTN2P_EMU128=0x11.so" "libblade_asa_BLADE_ATTN2P_EMU128=0x25.so"; do
  BLADE_LIB=$lib python scripts/attn_time.py --workload wan --calls 50 --blocks 3 >> $P/wan.jsonl 2>&1
done
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_EMU64=0x00.so" "libblade_asa_BLADE_ATTN2P_EMU64=0x11.so" "libblade_asa_BLADE_ATTN2P_EMU64=0x25.so" "libblade_asa_BLADE_ATTN2P_EMU64=0x55.so"; do
  BLADE_LIB=$lib python scripts/attn_time.py --workload cog --calls 50 --blocks 3 >> $P/cog.jsonl 2>&1
done
done
cat $P/wan.jsonl $P/cog.jsonl
