for lib in libblade_asa_BLADE_ATTN2_TRACE.so libblade_asa_BLADE_ATTN2_TRACE_BLADE_ATTN2_SKIP_SOFTMAX.so; do
 for wl in cog wan; do
  echo "== $lib $wl"
  BLADE_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --steps 12 --warmup 3 --workload $wl --attn pair 2>&1 >/dev/null | head -30
 done
done
