mkdir -p gpurun_out/r02tr
OUT=gpurun_out/r02tr
for v in TRACE_BLADE_ATTN2_SKIP_SOFTMAX_BLADE_ATTN2_SKIP_LOAD TRACE_BLADE_ATTN2_SKIP_SOFTMAX TRACE; do
  BLADE_LIB=libblade_asa_BLADE_ATTN2_$v.so timeout 300 python scripts/attn_time.py --workload wan --calls 5 --blocks 1 > $OUT/wan_$v.txt 2>&1
done
head -20 $OUT/*.txt
