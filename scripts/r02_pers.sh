# Persistent pair kernel (AUTO): quick parity first (short timeouts), then the suite and A/B.
mkdir -p gpurun_out/r02pers2
OUT=gpurun_out/r02pers2
timeout 240 python -m pytest tests/test_gpu_fused.py -q -x -k persistent > $OUT/pytest_quick.log 2>&1; rc=$?; tail -3 $OUT/pytest_quick.log
if [ $rc -ne 0 ]; then echo "quick test failed rc=$rc"; exit 1; fi
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for rep in 1 2 3; do
  for lib in libblade_asa.so libblade_asa_BLADE_ATTN2P_OFF.so; do
    for wl in wan cog; do
      BLADE_LIB=$lib timeout 60 python scripts/attn_time.py --workload $wl --blocks 3 >> $OUT/ab.jsonl 2>&1
      BLADE_LIB=$lib timeout 60 python scripts/attn_time.py --workload $wl --blocks 3 --fused >> $OUT/ab.jsonl 2>&1
    done
  done
done
for lib in libblade_asa.so libblade_asa_BLADE_ATTN2P_OFF.so; do
  BLADE_LIB=$lib timeout 60 python scripts/attn_time.py --workload wan --blocks 3 --fused --tau 0.9 >> $OUT/ab.jsonl 2>&1
done
cat $OUT/ab.jsonl
