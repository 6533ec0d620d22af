set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for c in 0 1 2 3 6; do timeout 300 python bench.py --no-cpu --steps 50 --e2e-chunk $c 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk $c', d['ms_per_step'], d['e2e'])"; done
timeout 600 python scripts/sweep.py --steps 10 > gpurun_out/sweep_wan.jsonl 2> gpurun_out/sweep.err; cat gpurun_out/sweep_wan.jsonl | cut -c1-400
timeout 900 python bench.py --workload wan_stack --steps 3 --warmup 3 > gpurun_out/stack1.json 2> gpurun_out/stack1.err; cat gpurun_out/stack1.json; tail -3 gpurun_out/stack1.err
