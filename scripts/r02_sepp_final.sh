# decoupled P for d = 64 as the default: GPU suite, sanitizers, bench lines
mkdir -p gpurun_out/r02sf
P=gpurun_out/r02sf
timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo "rc=$?" >> $P/pytest_gpu.log
tail -3 $P/pytest_gpu.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tests/tools/sanitize_cases.py > $P/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $P/sanitizer_$tool.log
  tail -2 $P/sanitizer_$tool.log
done
python bench.py --workload cog --no-extra --no-cpu > $P/bench_cog.json 2> $P/bench_cog.err
python bench.py --steps 20 --warmup 5 --no-cpu > $P/bench_wan.json 2> $P/bench_wan.err
cat $P/bench_cog.json | head -c 600; echo; cat $P/bench_wan.json | head -c 400
