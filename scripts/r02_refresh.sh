# Round-2 refresh on one B200: full GPU suite, smoke, bench lines, launch lists,
# pipe counters and one ncu --set full capture (copied into profiles/ by hand).
mkdir -p gpurun_out/r02r
P=gpurun_out/r02r
python -c "import __graft_entry__ as g; g.build()" > $P/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $P/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > $P/bench_wan.json 2> $P/bench_wan.err
python bench.py --impl reference --steps 20 --warmup 5 > $P/bench_ref.json 2> $P/bench_ref.err
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_wan.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_cog.csv $B --workload cog > /dev/null 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_wan.csv $B > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_cog.csv $B --workload cog > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2 -s 2 -c 1 -o $P/full_wan_attn -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:probe2 -s 2 -c 1 -o $P/full_wan_probe -f $B > /dev/null 2>&1
ls -la $P
