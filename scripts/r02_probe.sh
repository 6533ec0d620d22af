# tcgen05 probe for every k / N_b (R passes): mask GPU tests; MMA skeleton microbenchmark.
mkdir -p gpurun_out/r02p
OUT=gpurun_out/r02p
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
./scripts/mma_issue_bench.bin > $OUT/mma_issue_bench.txt 2>&1
python scripts/mask_time.py --workload wan --configs keep51,tau0.9 > $OUT/mask_wan.txt 2>&1
python scripts/mask_time.py --workload cog --configs keep25 > $OUT/mask_cog.txt 2>&1
cat $OUT/mma_issue_bench.txt $OUT/mask_wan.txt $OUT/mask_cog.txt
