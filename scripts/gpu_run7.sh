mkdir -p gpurun_out
for lib in libblade_asa.so libblade_asa_BLADE_ATTN2_SKIP_SOFTMAX.so libblade_asa_BLADE_ATTN2_SKIP_LOAD.so "libblade_asa_BLADE_ATTN2_EMU_MASK=0x55.so"; do
  for wl in wan cog; do
    BLADE_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --workload $wl --attn pair > gpurun_out/b7.json 2>&1
    python -c "import json; d=json.load(open('gpurun_out/b7.json')); print('$lib $wl', round(d['ms_attn'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b7.json
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc2_kernel -s 2 -c 1 -o gpurun_out/attn2_wan -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --attn pair > gpurun_out/ncu7.log 2>&1
