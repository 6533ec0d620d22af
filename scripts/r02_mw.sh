# Warp-collective tcgen05 issue + split-softmax kernels: GPU suite, 4-way A/B.
mkdir -p gpurun_out/r02mw
OUT=gpurun_out/r02mw
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
L="libblade_asa.so libblade_asa_BLADE_MMA_WARP=0.so libblade_asa_BLADE_ATTN1S_OFF_BLADE_ATTN2S_OFF.so libblade_asa_BLADE_MMA_WARP=0_BLADE_ATTN1S_OFF_BLADE_ATTN2S_OFF.so"
for rep in 1 2; do
  for lib in $L; do
    for wl in cog wan; do
      BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload $wl --blocks 3 >> $OUT/ab.jsonl 2>&1
    done
  done
done
cat $OUT/ab.jsonl
