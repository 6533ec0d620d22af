mkdir -p gpurun_out/r02c
OUT=gpurun_out/r02c
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
tail -3 $OUT/pytest_gpu.log
python scripts/mask_time.py --workload wan > $OUT/mask_wan.jsonl 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $OUT/mask_cog.jsonl 2>&1
cat $OUT/mask_wan.jsonl $OUT/mask_cog.jsonl
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"refine|sample" -c 8 --csv --log-file $OUT/refine_ncu.csv python scripts/mask_time.py --workload wan --steps 2 --configs keep51,tau0.95 > /dev/null 2>&1
python bench.py --steps 20 --no-extra --no-cpu --no-e2e > $OUT/bench.json 2>&1
