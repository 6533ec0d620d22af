mkdir -p gpurun_out/r02bwd
P=gpurun_out/r02bwd
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_BWD_EMU_MASK=0x00.so" "libblade_asa_BLADE_BWD_EMU_MASK=0x02.so" "libblade_asa_BLADE_BWD_EMU_MASK=0x10.so" "libblade_asa_BLADE_BWD_EMU_MASK=0x11.so" "libblade_asa_BLADE_BWD_EMU_MASK=0x22.so"; do
  echo "$lib cog $(BLADE_LIB=$lib python scripts/bench_bwd.py --workload cog | grep ms_bwd | cut -c1-80)" >> $P/bwd.txt
  echo "$lib wan $(BLADE_LIB=$lib python scripts/bench_bwd.py | grep ms_bwd | cut -c1-80)" >> $P/bwd.txt
done
done
cat $P/bwd.txt
