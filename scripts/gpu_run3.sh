set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gt.py tests/test_gpu_host_pipeline.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_gt.log; tail -30 gpurun_out/pytest_gt.log
for c in 0 1 2 3 6; do timeout 300 python bench.py --no-cpu --steps 50 --e2e-chunk $c 2>/dev/null > gpurun_out/e2e_chunk$c.json; python -c "import json; d=json.load(open('gpurun_out/e2e_chunk$c.json')); print('chunk $c', d['ms_per_step'], d['e2e'])"; done
timeout 300 python bench.py --no-cpu --no-e2e --variant asa_gt > gpurun_out/bench_gt.json 2>&1; cat gpurun_out/bench_gt.json
./scripts/fp64_bench.bin > gpurun_out/fp64_bench.txt 2>&1; cat gpurun_out/fp64_bench.txt
