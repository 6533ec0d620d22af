# Speculative exponentials in the pair kernel: GPU suite, A/B, trace.
mkdir -p gpurun_out/r02spec
OUT=gpurun_out/r02spec
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
for rep in 1 2 3; do
  for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2_SPEC_EXP=0.so"; do
    for wl in wan cog; do
      BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload $wl --blocks 3 >> $OUT/ab.jsonl 2>&1
    done
  done
done
BLADE_LIB=libblade_asa_BLADE_ATTN2_TRACE.so timeout 300 python scripts/attn_time.py --workload wan --calls 5 --blocks 1 > $OUT/trace_wan.txt 2>&1
cat $OUT/ab.jsonl; head -16 $OUT/trace_wan.txt
