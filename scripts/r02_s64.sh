# d=64 column-split attention kernel: GPU suite, A/B vs the pair kernel.
mkdir -p gpurun_out/r02s64b
OUT=gpurun_out/r02s64b
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
for rep in 1 2; do
  for lib in libblade_asa.so libblade_asa_BLADE_ATTN2S_OFF.so; do
    BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload cog --blocks 3 >> $OUT/ab.jsonl 2>&1
    BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload cog --fused --blocks 3 >> $OUT/ab.jsonl 2>&1
  done
done
ncu --set full --import-source on --clock-control none -k regex:attn_tc2s -s 2 -c 1 -o $OUT/full_s64 -f python scripts/attn_time.py --workload cog --calls 3 --blocks 1 > /dev/null 2>&1
cat $OUT/ab.jsonl
