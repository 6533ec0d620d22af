set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gt.py -x -q -k "attention or gt or end_to_end or invariants" 2>&1 | tail -15 > gpurun_out/pytest5.log; tail -15 gpurun_out/pytest5.log
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN_SPLIT=1.so"; do
  for wl in wan cog; do
    BLADE_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --workload $wl > gpurun_out/b5_${wl}_${lib}.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/b5_${wl}_${lib}.json')); print('$lib $wl', round(d['ms_attn'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
