mkdir -p gpurun_out/r02f
OUT=gpurun_out/r02f
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
tail -15 $OUT/pytest_gpu.log
python scripts/mask_time.py --workload wan > $OUT/mask_wan.jsonl 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $OUT/mask_cog.jsonl 2>&1
BLADE_LIB=libblade_asa_BLADE_PROBE_V1.so python scripts/mask_time.py --workload wan --configs keep51 > $OUT/mask_wan_v1.jsonl 2>&1
cat $OUT/mask_*.jsonl
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none -c 10 --csv --log-file $OUT/mask_ncu.csv python scripts/mask_time.py --workload wan --steps 1 --configs keep51,tau0.95 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:probe -c 1 -o $OUT/probe2 -f python scripts/mask_time.py --workload wan --steps 1 --configs keep51 > /dev/null 2>&1
BLADE_LIB=libblade_asa_BLADE_PROBE_V1.so ncu --set full --import-source on --clock-control none -k regex:probe -c 1 -o $OUT/probe_v1 -f python scripts/mask_time.py --workload wan --steps 1 --configs keep51 > /dev/null 2>&1
python bench.py --steps 20 --no-extra --no-cpu > $OUT/bench.json 2>&1
