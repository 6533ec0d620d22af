# Round-2 evidence: tensor / XU / shared / TMA pipe counters of the step's kernels,
# compute-sanitizer on tiny and odd N, plus the baseline bench lines.
mkdir -p gpurun_out/r02
OUT=gpurun_out/r02
python bench.py --steps 20 --warmup 5 > $OUT/bench_wan_20.json 2> $OUT/bench_wan_20.err
python bench.py --steps 200 --warmup 5 --no-cpu > $OUT/bench_wan_200.json 2> $OUT/bench_wan_200.err
python bench.py --workload cog --steps 50 --no-cpu > $OUT/bench_cog.json 2> $OUT/bench_cog.err
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $OUT/pipes_wan.csv $B > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $OUT/pipes_cog.csv $B --workload cog > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $OUT/pipes_wan_tau95.csv $B --tau-mode --tau 0.95 > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tests/tools/sanitize_cases.py > $OUT/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_$tool.log
done
ls -la $OUT
