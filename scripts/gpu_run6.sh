set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gt.py -x -q -k "pair" 2>&1 | tail -15 > gpurun_out/pytest6.log; tail -15 gpurun_out/pytest6.log
for impl in tcgen05 pair; do
  for wl in wan cog; do
    timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --workload $wl --attn $impl > gpurun_out/b6_${wl}_${impl}.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/b6_${wl}_${impl}.json')); print('$impl $wl', round(d['ms_attn'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/b6_${wl}_${impl}.json
  done
done
