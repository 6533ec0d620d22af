mkdir -p gpurun_out/r02qpf
OUT=gpurun_out/r02qpf
timeout 240 python -m pytest tests/test_gpu_fused.py -q -x -k persistent > $OUT/pytest_quick.log 2>&1; rc=$?; tail -n 2 $OUT/pytest_quick.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2 3; do
  for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_QPREFETCH=0.so"; do
    for wl in wan cog; do
      BLADE_LIB=$lib timeout 60 python scripts/attn_time.py --workload $wl --blocks 2 >> $OUT/ab.jsonl 2>&1
    done
  done
done
cat $OUT/ab.jsonl
