mkdir -p gpurun_out/r02mf4
OUT=gpurun_out/r02mf4
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for rep in 1 2; do
  for lib in libblade_asa.so libblade_asa_BLADE_MASK_UNFUSED.so "libblade_asa_BLADE_MF_SELWARPS=2.so"; do
    echo "$lib $(BLADE_LIB=$lib timeout 300 python scripts/mask_time.py --workload wan --configs keep51,tau0.9)" >> $OUT/mask.txt 2>&1
    echo "$lib $(BLADE_LIB=$lib timeout 300 python scripts/mask_time.py --workload cog --configs keep25,tau0.9)" >> $OUT/mask.txt 2>&1
    BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload wan --fused --blocks 3 >> $OUT/fused.jsonl 2>&1
    BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload cog --fused --blocks 3 >> $OUT/fused.jsonl 2>&1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_wan.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_cog.csv python bench.py --workload cog --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1
cat $OUT/mask.txt $OUT/fused.jsonl
