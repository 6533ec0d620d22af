# Chunked P hand-off: parity of the attention tests, A/B of 1 / 2 / 4 chunks, trace.
mkdir -p gpurun_out/r02pc
OUT=gpurun_out/r02pc
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or fused or gt or edges or headline" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
L="libblade_asa.so libblade_asa_BLADE_ATTN2_PCHUNKS=1.so libblade_asa_BLADE_ATTN2_PCHUNKS=2.so"
for rep in 1 2 3; do
  for lib in $L; do
    for wl in wan cog; do
      BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload $wl --blocks 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
    done
  done
done
BLADE_LIB=libblade_asa_BLADE_ATTN2_TRACE.so timeout 300 python scripts/attn_time.py --workload wan --calls 5 --blocks 1 > $OUT/trace_wan.txt 2>&1
BLADE_LIB=libblade_asa_BLADE_ATTN2_TRACE.so timeout 300 python scripts/attn_time.py --workload cog --calls 5 --blocks 1 > $OUT/trace_cog.txt 2>&1
cat $OUT/ab.jsonl
