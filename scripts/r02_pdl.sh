# PDL chain check: GPU suite, mask timings, a bench line
mkdir -p gpurun_out/r02pdl
P=gpurun_out/r02pdl
python -c "import __graft_entry__ as g; g.build()" > $P/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo "rc=$?" >> $P/pytest_gpu.log
tail -3 $P/pytest_gpu.log
python scripts/mask_time.py --workload wan > $P/mask_wan.jsonl 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $P/mask_cog.jsonl 2>&1
cat $P/mask_wan.jsonl $P/mask_cog.jsonl
python bench.py --steps 20 --warmup 5 --no-cpu > $P/bench.json 2> $P/bench.err
cat $P/bench.json
