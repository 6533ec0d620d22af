# Attention A/B on one box: skip-experiments, exponential-emulation masks, trace.
mkdir -p gpurun_out/r02ab
OUT=gpurun_out/r02ab
L="libblade_asa.so libblade_asa_BLADE_ATTN2_SKIP_SOFTMAX.so libblade_asa_BLADE_ATTN2_SKIP_LOAD.so libblade_asa_BLADE_ATTN2_SKIP_SOFTMAX_BLADE_ATTN2_SKIP_LOAD.so libblade_asa_BLADE_ATTN2_EMU_MASK=0x01.so libblade_asa_BLADE_ATTN2_EMU_MASK=0x11.so libblade_asa_BLADE_ATTN2_EMU_MASK=0x55.so"
for rep in 1 2; do
  for lib in $L; do
    for wl in wan cog; do
      BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload $wl >> $OUT/ab.jsonl 2>> $OUT/ab.err
    done
  done
done
BLADE_LIB=libblade_asa_BLADE_ATTN2_TRACE.so timeout 300 python scripts/attn_time.py --workload wan --calls 5 --blocks 1 > $OUT/trace_wan.txt 2>&1
BLADE_LIB=libblade_asa_BLADE_ATTN2_TRACE.so timeout 300 python scripts/attn_time.py --workload cog --calls 5 --blocks 1 > $OUT/trace_cog.txt 2>&1
cat $OUT/ab.jsonl
