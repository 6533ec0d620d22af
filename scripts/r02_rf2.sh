# Refine: one-pass combine + warp-level fp64 reselection; phase timings; pipe counters at tau 0.95.
mkdir -p gpurun_out/r02rf2
OUT=gpurun_out/r02rf2
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
BLADE_LIB=libblade_asa_BLADE_RF_TIMING.so timeout 300 python scripts/mask_time.py --workload wan --configs keep51,tau0.9,tau0.95 > $OUT/rf_timing.txt 2>&1
python scripts/mask_time.py --workload wan --configs keep51,tau0.9,tau0.95 > $OUT/mask_wan.txt 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $OUT/mask_cog.txt 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M -k regex:refine --clock-control none -c 2 --csv --log-file $OUT/refine_ncu.csv python scripts/mask_time.py --workload wan --steps 1 --configs tau0.95 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:refine -s 1 -c 1 -o $OUT/refine95 -f python scripts/mask_time.py --workload wan --steps 1 --configs tau0.95 > /dev/null 2>&1
cat $OUT/rf_timing.txt $OUT/mask_wan.txt $OUT/mask_cog.txt
