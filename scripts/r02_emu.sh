mkdir -p gpurun_out/r02h
OUT=gpurun_out/r02h
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_PROBE_EMU=0x11.so" "libblade_asa_BLADE_PROBE_EMU=0x49.so" "libblade_asa_BLADE_PROBE_EMU=0x55.so" "libblade_asa_BLADE_PROBE_EMU=0x5b.so" libblade_asa_BLADE_PROBE_V1.so; do
  echo "$lib $(BLADE_LIB=$lib python scripts/mask_time.py --workload wan --configs keep51 --steps 30)" >> $OUT/emu.txt
done
done
cat $OUT/emu.txt
for lib in libblade_asa.so "libblade_asa_BLADE_PROBE_EMU=0x49.so"; do
BLADE_LIB=$lib ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed -k regex:probe --clock-control none -c 3 --csv --log-file "$OUT/emu_$lib.csv" python scripts/mask_time.py --workload wan --configs keep51 --steps 2 > /dev/null 2>&1
done
