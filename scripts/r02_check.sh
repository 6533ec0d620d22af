# Round-2 GPU check: new tests, the full gpu suite, bench lines, synccheck.
mkdir -p gpurun_out/r02b
OUT=gpurun_out/r02b
timeout 1500 python -m pytest tests -m gpu -q -x -k "headline or shard or many_ctas" > $OUT/pytest_new.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
tail -3 $OUT/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tests/tools/sanitize_cases.py > $OUT/sanitizer_synccheck.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_synccheck.log
ls -la $OUT
