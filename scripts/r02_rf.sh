mkdir -p gpurun_out/r02g
OUT=gpurun_out/r02g
BLADE_LIB=libblade_asa_BLADE_RF_TIMING.so python scripts/mask_time.py --workload wan --configs keep51,tau0.95 > $OUT/rf_wan.txt 2>&1
cat $OUT/rf_wan.txt
ncu --set full --import-source on --clock-control none -k regex:"refine" -s 1 -c 1 -o $OUT/refine51 -f python scripts/mask_time.py --workload wan --steps 2 --configs keep51 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"sample" -s 1 -c 1 -o $OUT/sample -f python scripts/mask_time.py --workload wan --steps 2 --configs keep51 > /dev/null 2>&1
ls $OUT
