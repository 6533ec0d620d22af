mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gt.py -x -q -k "attention or gt" 2>&1 | tail -3
for lib in libblade_asa.so libblade_asa_BLADE_ATTN2_SKIP_SOFTMAX.so; do
  for impl in tcgen05 pair; do
  for wl in wan cog; do
    BLADE_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --workload $wl --attn $impl > gpurun_out/b8.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/b8.json')); print('$lib $impl $wl', round(d['ms_attn'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b8.json
  done
  done
done
