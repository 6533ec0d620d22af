set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_wan.json 2> gpurun_out/bench_wan.err; cat gpurun_out/bench_wan.json; tail -5 gpurun_out/bench_wan.err
timeout 600 python bench.py --workload cog --no-cpu > gpurun_out/bench_cog.json 2> gpurun_out/bench_cog.err; cat gpurun_out/bench_cog.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_wan.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu $?
